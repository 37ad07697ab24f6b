"""The result printer at SURVEY.md 8(f) scale: C5's 4.17 M-term determinant
(through the public API on the GPU) formatted by the native host formatter
equals the oracle restatement of the reference's format_polynomial
(parsing.py:197-225) byte for byte."""

import hashlib
import time

import pytest

from oracle import polydet_oracle as O

pytestmark = pytest.mark.gpu


def test_c5_result_text(cuda):
    from paper_2010_12117_b200 import format_polynomial, run, workloads

    m, cfg = workloads.c5()
    result = run(m, cfg)
    terms = result.terms()
    assert len(terms) == 161 ** 3
    t0 = time.perf_counter()
    text = format_polynomial(terms, result.axis_vars)
    t_native = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = O.format_polynomial(terms, result.axis_vars)
    t_oracle = time.perf_counter() - t0
    assert hashlib.sha256(text.encode()).hexdigest() == hashlib.sha256(want.encode()).hexdigest()
    assert text == want
    print("C5 text: %d terms, %.0f MB, native %.2f s, oracle %.2f s" % (len(terms), len(text) / 1e6, t_native,
                                                                     t_oracle))
