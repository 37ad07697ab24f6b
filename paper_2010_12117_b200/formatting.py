"""Canonical polynomial text -- drop-in for the reference's `format_polynomial`
(parsing.py:197-225), the printer of a determinant result (cli.py:61-83).

Same output byte for byte: terms in graded lexicographic order, highest
first; `x`, `x^e` factors joined by `*`; `|c|*` unless |c| = 1; ` + ` / ` - `
between terms; `0` for no terms.  The sort, the decimal digits of the
coefficients (hundreds of bits each for C5's 4.17 M terms) and the string
assembly run in the native host module (`_pdb_host.format_terms`,
csrc/host_ints.cpp), multi-threaded.  A `CoeffTensor` may be passed in place
of its `terms()`.
"""

from __future__ import annotations

import os
from collections.abc import Mapping

from . import native
from .layout import CoeffTensor, normalize_terms


def _threads() -> int:
    return max(1, min(os.cpu_count() or 1, 32))


def format_polynomial(terms, variables) -> str:
    """Canonical text: graded lexicographic order, highest terms first."""
    variables = tuple(str(v) for v in variables)
    host = native.host_module()
    if isinstance(terms, CoeffTensor) and len(terms.shape) == len(variables):
        # straight from the dense coefficients: no terms() dict of 10^6-10^7 tuples
        try:
            return host.format_dense(terms.coeffs, tuple(int(n) for n in terms.shape), variables, _threads())
        except TypeError:
            pass
    if isinstance(terms, CoeffTensor):
        terms = terms.terms()
    if isinstance(terms, dict) and type(terms) is dict:
        try:
            if all(len(e) == len(variables) for e in terms):
                return host.format_terms(terms, variables, _threads())
        except TypeError:
            pass   # keys/values that are not plain ints: normalise as the reference does
    norm = normalize_terms(terms.items() if isinstance(terms, Mapping) else terms)
    k = len(variables)
    if all(len(e) == k for e in norm):
        return host.format_terms(norm, variables, _threads())
    # exponent tuples of another arity: the reference zips names and exponents
    # (extra exponents still count in the degree); pad/truncate to the names
    # for the text and keep the degree of the full tuple in the order
    return _format_mismatched(norm, variables)


def _format_mismatched(norm: dict, variables: tuple) -> str:
    if not norm:
        return "0"
    ordered = sorted(norm.items(), key=lambda item: (sum(item[0]), item[0]), reverse=True)
    pieces = []
    for index, (exps, coeff) in enumerate(ordered):
        parts = [v if e == 1 else "%s^%d" % (v, e) for v, e in zip(variables, exps) if e >= 1]
        mag = abs(coeff)
        if not parts:
            text = str(mag)
        else:
            body = "*".join(parts)
            text = body if mag == 1 else "%d*%s" % (mag, body)
        if index == 0:
            pieces.append("-" + text if coeff < 0 else text)
        else:
            pieces.append(("- " if coeff < 0 else "+ ") + text)
    return " ".join(pieces)
