"""Pin the CPU oracle to the reference: every golden vector produced by the
reference implementation (tests/golden/make_golden.py) must be reproduced by
oracle/polydet_oracle.py.  CPU only."""

import numpy as np
import pytest

from helpers import golden
from oracle import polydet_oracle as O


def test_oracle_ntt_matches_reference():
    for case in golden("ntt.json"):
        p, _c, q, w = case["prime"]
        shape = tuple(case["shape"])
        if p > O.INT64_SAFE:
            continue
        fwd = O.ntt_multi(case["input"], shape, p, w, q)
        inv = O.ntt_multi(case["input"], shape, p, w, q, inverse=True)
        assert fwd.tolist() == case["forward"], (p, shape)
        assert inv.tolist() == case["inverse"], (p, shape)


def test_oracle_det_matches_reference():
    for case in golden("det.json"):
        p = case["prime"][0]
        grids = [np.array(g, dtype=np.int64) for g in case["grids"]]
        out = O.det_grid(grids, case["r"], p, case["entry_ids"])
        assert out.tolist() == case["expected"], case["note"]


def test_oracle_condense_trail_matches_reference():
    """Pivot values, columns, sign flags and the determinant of the reference's
    condensation (golden condense.json)."""
    for case in golden("condense.json"):
        det, records = O.condense_trail(case["rows"], case["prime"][0])
        assert det == case["det"], case["note"]
        assert [list(rec) for rec in records] == case["records"], case["note"]


def test_oracle_det_chunk_and_thread_invariance():
    case = next(c for c in golden("det.json") if c["r"] == 5)
    grids = [np.array(g, dtype=np.int64) for g in case["grids"]]
    p = case["prime"][0]
    base = O.det_grid(grids, 5, p)
    for chunk in (1, 7, 100):
        for workers in (1, 3):
            assert O.det_grid(grids, 5, p, chunk=chunk, workers=workers).tolist() == base.tolist()


def test_oracle_crt_matches_reference():
    for case in golden("crt.json"):
        out = O.crt_combine(case["residues"], case["primes"])
        assert [str(v) for v in out] == case["expected"]


@pytest.mark.parametrize("limit", [25])
def test_oracle_end_to_end_matches_reference(limit):
    from paper_2010_12117_b200 import layout, planner

    for case in golden("runs.json")[:limit]:
        m = layout.PolyMatrix.from_dict(case["input"])
        cfg = planner.PipelineConfig(**case["config"])
        pl = planner.plan(m, cfg)
        assert pl.digest() == case["digest"]
        terms = [t.terms() for t in m.unique_entries]
        coeffs, _ = O.run_pipeline(terms, m.entry_ids, m.r, pl.shape,
                                   [(s.p, s.omega, s.q) for s in pl.primes])
        got = layout.CoeffTensor(pl.shape, tuple(coeffs), pl.variables).terms()
        want = {tuple(e): c for e, c in case["terms"]}
        assert got == want, case["name"]
