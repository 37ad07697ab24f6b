"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the dev container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--c3]

It imports the reference package read-only from /root/reference/pkg/src and
writes small JSON fixtures next to this file.  Nothing on the GPU box reads
/root/reference; the tests read these committed files instead.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import random
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(1, str(REPO))

import numpy as np  # noqa: E402
import polydet as ref  # noqa: E402  (the reference)
import polydet.tensor  # noqa: E402,F401
import polydet.workspace  # noqa: E402,F401
from oracles import random_matrix_terms, random_terms  # noqa: E402  (reference test oracles)

from paper_2010_12117_b200 import workloads  # noqa: E402  (only for the config recipes)


def _write(name, obj):
    path = HERE / name
    path.write_text(json.dumps(obj, separators=(",", ":")))
    print("wrote", path, path.stat().st_size, "bytes")


def _ref_matrix(m):
    return ref.PolyMatrix.from_dict(m.to_dict())


def _ref_cfg(cfg, **kw):
    return ref.PipelineConfig(prime_start=cfg.prime_start, min_primes=cfg.min_primes, **kw)


def _terms_json(terms):
    return [[list(e), int(c)] for e, c in sorted(terms.items())]


def plans():
    out = {}
    cases = {
        "C1": workloads.c1(), "C2": workloads.c2(), "C2w": workloads.c2(True),
        "C3": workloads.c3(), "C5": workloads.c5(),
        "C4_3src_T5T7_m": workloads.harmonic(3, (5, 7), True),
        "C4_4src_T5T11_m": workloads.harmonic(4, (5, 11), True),
    }
    for name, (m, cfg) in cases.items():
        pl = ref.plan(_ref_matrix(m), _ref_cfg(cfg))
        out[name] = {"digest": pl.digest(), "plan": pl.to_dict(),
                     "input_digest": ref.workspace.digest_of(_ref_matrix(m).to_dict())}
    _write("plans.json", out)


def primes():
    out = {
        "root_17_16": ref.find_root_of_order(17, 16),
        "root_2013265921_2^27": ref.find_root_of_order(2013265921, 2**27),
        "q6_first3": [[s.p, s.c, s.q, s.omega] for s in ref.find_fourier_primes(6, 1, 10**9, min_count=3)],
        "q8_first3": [[s.p, s.c, s.q, s.omega] for s in ref.find_fourier_primes(8, 1, 10**9, min_count=3)],
        "q0_small": [s.p for s in ref.find_fourier_primes(0, 1, 2, min_count=2)],
        "q0_big": [s.p for s in ref.find_fourier_primes(0, 1, 10**9, min_count=2)],
        "q30": [s.p for s in ref.find_fourier_primes(30, 1, 2, min_count=1)],
        "q27_2e9": [[s.p, s.c, s.q, s.omega] for s in ref.find_fourier_primes(27, 1, 2 * 10**9, min_count=1)],
        "q26_start": [[s.p, s.c, s.q, s.omega] for s in ref.find_fourier_primes(26, 1, 1800000000, min_count=1)],
        "q10_set": [[s.p, s.c, s.q, s.omega] for st in (10**4, 10**6, 10**9)
                    for s in ref.find_fourier_primes(10, 1, start=st, min_count=1)],
        "census": {str(k): v for k, v in ref.census((64, 128, 256, 512, 4096, 8192, 65536), 2000).counts.items()},
    }
    _write("primes.json", out)


def _spec_list():
    specs = [ref.find_fourier_primes(4, 1, start=97, min_count=1)[0]]
    specs += [ref.find_fourier_primes(10, 1, start=s, min_count=1)[0] for s in (10**4, 10**6, 10**9)]
    specs.append(ref.find_fourier_primes(27, 1, start=2 * 10**9, min_count=1)[0])
    specs.append(ref.find_fourier_primes(4, 1, start=2**30, min_count=1)[0])
    specs.append(ref.find_fourier_primes(13, 1, start=10**9, min_count=1)[0])
    return specs


def ntt_cases():
    rng = random.Random(11)
    cases = []
    for spec in _spec_list():
        table = ref.TwiddleTable(spec)
        shapes = [(), (1,), (2,), (4,), (8,), (16,), (4, 4), (2, 8, 4), (1, 4, 2), (16, 1, 2)]
        if spec.q >= 6:
            shapes += [(64,), (16, 16, 8), (32, 8), (4, 4, 4, 4), (2, 64)]
        if spec.q >= 10:
            shapes += [(1024,), (8, 128)]
        if spec.q >= 13:
            shapes += [(8192,), (4096, 2), (2, 2048)]
        for shape in shapes:
            size = int(np.prod(shape)) if shape else 1
            vals = [rng.randrange(spec.p) for _ in range(size)]
            names = tuple("v%d" % i for i in range(len(shape)))
            mt = ref.ModTensor(shape, np.array(vals, dtype=ref.tensor.residue_dtype(spec)), spec, names)
            fwd = ref.ntt_forward_multi(mt, table).residues.tolist()
            inv = ref.ntt_inverse_multi(mt, table).residues.tolist()
            cases.append({"prime": [spec.p, spec.c, spec.q, spec.omega], "shape": list(shape),
                          "input": vals, "forward": [int(v) for v in fwd], "inverse": [int(v) for v in inv]})
    _write("ntt.json", cases)


def det_cases():
    rng = random.Random(12)
    specs = _spec_list()
    cases = []

    def add(spec, r, mats, ids=None, k=None, note=""):
        nodes = len(mats)
        if ids is None:
            grids = [[mats[n][e // r][e % r] for n in range(nodes)] for e in range(r * r)]
        else:
            grids = [[mats[n][e] for n in range(nodes)] for e in range(k)]
        g = [np.array(x, dtype=ref.tensor.residue_dtype(spec)) for x in grids]
        out = ref.det_grid(g, r, spec, entry_ids=ids)
        cases.append({"prime": [spec.p, spec.c, spec.q, spec.omega], "r": r, "grids": grids,
                      "entry_ids": ids, "expected": [int(v) for v in out], "note": note})

    for spec in specs[:1] + specs[3:6]:
        p = spec.p
        for r in (1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24, 32, 40, 48, 64):
            nodes = 33 if r <= 16 else 9
            mats = [[[rng.randrange(p) for _ in range(r)] for _ in range(r)] for _ in range(nodes)]
            if r >= 2:
                mats[1][r - 1] = list(mats[1][0])                      # duplicate row -> 0
                mats[2][0] = [0] * r                                   # zero row -> 0
                mats[3][0][0] = 0                                      # zero leading pivot
                for i in range(r):                                     # strictly permuted pivots
                    mats[4][i] = [0] * (r - 1 - i) + [rng.randrange(1, p) for _ in range(i + 1)]
                mats[5] = [[rng.randrange(p) if rng.random() < 0.4 else 0 for _ in range(r)] for _ in range(r)]
                mats[6] = [[(i + j) % 2 * rng.randrange(p) for j in range(r)] for i in range(r)]
                mats[7] = [[int(i == j) for j in range(r)] for i in range(r)]
                mats[8] = [[0] * r for _ in range(r)]
            add(spec, r, mats, note="random+special r=%d" % r)
        # dedup ids: [[a, b], [b, a]]
        mats = [[rng.randrange(p), rng.randrange(p)] for _ in range(16)]
        add(spec, 2, mats, ids=[0, 1, 1, 0], k=2, note="dedup")
    # the permuted-pivot known answer (test_determinant.py:67-75) mod 97
    add(specs[0], 3, [[[0, 0, 2], [0, 3, 1], [4, 1, 5]]], note="permuted pivots")
    _write("det.json", cases)


def crt_cases():
    rng = random.Random(13)
    cases = []
    for count in (1, 2, 3, 7, 22, 23, 40):
        specs = ref.find_fourier_primes(6, 1, 10**9, min_count=count)
        product = 1
        for s in specs:
            product *= s.p
        half = product // 2
        vals = [rng.randint(-half + 1, half) for _ in range(40)] + [0, 1, -1, half, -half + 1]
        tensors = [ref.reduce_mod(ref.CoeffTensor((len(vals),), tuple(vals), ("x",)), s) for s in specs]
        out = ref.combine_tensor(tensors)
        assert list(out.coeffs) == vals
        cases.append({"primes": [s.p for s in specs],
                      "residues": [[int(v) for v in t.residues] for t in tensors],
                      "expected": [str(v) for v in out.coeffs]})
    # random residues (not from a known integer)
    specs = ref.find_fourier_primes(6, 1, 10**9, min_count=5)
    res = [[rng.randrange(s.p) for _ in range(64)] for s in specs]
    tensors = [ref.ModTensor((64,), np.array(r, dtype=np.int64), s, ("x",)) for r, s in zip(res, specs)]
    out = ref.combine_tensor(tensors)
    cases.append({"primes": [s.p for s in specs], "residues": res, "expected": [str(v) for v in out.coeffs]})
    _write("crt.json", cases)


def run_cases():
    cases = []
    rng = random.Random(20250808)
    for n in range(60):
        r = rng.randint(1, 5)
        vn = rng.randint(1, 3)
        d = rng.randint(0, 4)
        rows = random_matrix_terms(rng, r, vn, d, 100, 4)
        names = tuple("xyz"[:vn])
        m = ref.poly_matrix(rows, names)
        result, _, pl = ref.run_report(m)
        cases.append({"name": "ac3_%d" % n, "input": m.to_dict(), "config": {},
                      "digest": pl.digest(), "shape": list(result.shape),
                      "terms": _terms_json(result.terms())})
    for name, (m, cfg) in {"C1": workloads.c1(), "C2": workloads.c2(),
                           "C4_3src_T5T7_m": workloads.harmonic(3, (5, 7), True)}.items():
        rm = _ref_matrix(m)
        result, _, pl = ref.run_report(rm, _ref_cfg(cfg))
        cases.append({"name": name, "input": rm.to_dict(),
                      "config": {"prime_start": cfg.prime_start, "min_primes": cfg.min_primes},
                      "digest": pl.digest(), "shape": list(result.shape),
                      "terms": _terms_json(result.terms())})
    # univariate Sylvester demos (shape () results) and an order-8 dedup case
    for f, g, var, names in [({(2,): 1, (0,): 1}, {(1,): 1, (0,): 1}, "x", ("x",)),
                             ({(2,): 1, (0,): -1}, {(1,): 1, (0,): -1}, "x", ("x",)),
                             ({(4, 0, 0): 1, (1, 1, 0): 1, (0, 0, 1): 1},
                              {(4, 0, 0): 1, (2, 0, 1): 1, (0, 1, 0): 1}, "x", ("x", "u", "v"))]:
        m = ref.sylvester(f, g, names, var)
        result, _, pl = ref.run_report(m)
        cases.append({"name": "sylvester_%s" % len(cases), "input": m.to_dict(), "config": {},
                      "digest": pl.digest(), "shape": list(result.shape),
                      "terms": _terms_json(result.terms())})
    _write("runs.json", cases)


def workspace_case():
    """Artifact names + sha256s of a small checkpointed run (cross-resume pin)."""
    rng = random.Random(14)
    rows = random_matrix_terms(rng, 3, 2, 2, 25, 3)
    m = ref.poly_matrix(rows, ("x", "y"))
    with tempfile.TemporaryDirectory() as tmp:
        units = []
        ref.run(m, ref.PipelineConfig(progress=units.append), workspace=Path(tmp) / "ws")
        manifest = (Path(tmp) / "ws" / "manifest").read_text().splitlines()
        files = {p.name: hashlib.sha256(p.read_bytes()).hexdigest()
                 for p in sorted((Path(tmp) / "ws").iterdir())}
    _write("workspace.json", {"input": m.to_dict(), "units": units, "manifest": manifest, "files": files})


def wide_cases():
    """Primes >= 2^31: the reference's int64 (p <= 3.04e9) and object-dtype
    (p up to 2^62) paths -- NTTs, determinants, a mixed-prime CRT, end-to-end
    runs at prime_start = 2^61 and a checkpointed workspace's file hashes
    (reference tests: test_transform.py:221-230, test_determinant.py:105-114,
    test_crt.py:147-153, test_pipeline.py:149-153, test_workspace.py:179-189)."""
    rng = random.Random(15)
    out = {"ntt": [], "det": [], "crt": [], "runs": []}
    specs = [ref.find_fourier_primes(4, 1, start=2**61, min_count=1)[0],       # object dtype
             ref.find_fourier_primes(10, 1, start=2**31 + 1, min_count=1)[0],  # int64, > 2^31
             ref.find_fourier_primes(6, 1, start=3 * 10**9, min_count=1)[0]]    # object, < 2^32
    for spec in specs:
        table = ref.TwiddleTable(spec)
        dt = ref.tensor.residue_dtype(spec)
        for shape in [(16,), (4, 4), (2, 8, 1), (1,), ()]:
            size = int(np.prod(shape)) if shape else 1
            vals = [rng.randrange(spec.p) for _ in range(size)]
            mt = ref.ModTensor(shape, np.array(vals, dtype=dt), spec, tuple("v%d" % i for i in range(len(shape))))
            out["ntt"].append({"prime": [spec.p, spec.c, spec.q, spec.omega], "shape": list(shape), "input": vals,
                               "forward": [int(v) for v in ref.ntt_forward_multi(mt, table).residues.tolist()],
                               "inverse": [int(v) for v in ref.ntt_inverse_multi(mt, table).residues.tolist()],
                               "dtype": str(dt)})
        for r in (1, 2, 3, 4, 6, 9, 12):
            nodes = 12
            mats = [[[rng.randrange(spec.p) for _ in range(r)] for _ in range(r)] for _ in range(nodes)]
            if r >= 2:
                mats[1][r - 1] = list(mats[1][0])
                mats[2][0] = [0] * r
                mats[3][0][0] = 0
            grids = [[mats[n][e // r][e % r] for n in range(nodes)] for e in range(r * r)]
            g = [np.array(x, dtype=dt) for x in grids]
            det = ref.det_grid(g, r, spec)
            out["det"].append({"prime": [spec.p, spec.c, spec.q, spec.omega], "r": r, "grids": grids,
                               "expected": [int(v) for v in det], "dtype": str(det.dtype)})
    for start in (2**61, 2**31 + 1):
        cs = ref.find_fourier_primes(6, 1, start, min_count=3) + ref.find_fourier_primes(6, 1, 10**9, min_count=2)
        product = 1
        for sp in cs:
            product *= sp.p
        half = product // 2
        vals = [rng.randint(-half + 1, half) for _ in range(30)] + [0, 1, -1, half, -half + 1]
        tensors = [ref.reduce_mod(ref.CoeffTensor((len(vals),), tuple(vals), ("x",)), sp) for sp in cs]
        res = ref.combine_tensor(tensors)
        assert list(res.coeffs) == vals
        out["crt"].append({"primes": [sp.p for sp in cs], "residues": [[int(v) for v in t.residues] for t in tensors],
                           "expected": [str(v) for v in res.coeffs]})
    for n in range(6):
        r = rng.randint(1, 4)
        vn = rng.randint(1, 2)
        rows = random_matrix_terms(rng, r, vn, rng.randint(0, 3), 50, 3)
        m = ref.poly_matrix(rows, tuple("xy"[:vn]))
        result, _, pl = ref.run_report(m, ref.PipelineConfig(prime_start=2**61))
        out["runs"].append({"name": "wide_%d" % n, "input": m.to_dict(), "config": {"prime_start": 2**61},
                            "digest": pl.digest(), "shape": list(result.shape),
                            "terms": _terms_json(result.terms())})
    rows = random_matrix_terms(random.Random(13), 3, 2, 2, 25, 3)
    m = ref.poly_matrix(rows, ("x", "y"))
    with tempfile.TemporaryDirectory() as tmp:
        units = []
        ref.run(m, ref.PipelineConfig(prime_start=2**61, progress=units.append), workspace=Path(tmp) / "ws")
        files = {q.name: hashlib.sha256(q.read_bytes()).hexdigest() for q in sorted((Path(tmp) / "ws").iterdir())}
    out["workspace"] = {"input": m.to_dict(), "units": units, "files": files}
    _write("wide.json", out)


def c5_det_samples(n_nodes=24):
    """DET values of C5 at sampled nodes for primes 0 and 22 (direct evaluation).

    Entry values at node (a,b,c) are evaluated directly (the reference tests
    pin ntt_forward_multi == direct evaluation, test_transform.py:133-158),
    then the reference's det_grid takes the determinant.
    """
    m, cfg = workloads.c5()
    rm = _ref_matrix(m)
    pl = ref.plan(rm, _ref_cfg(cfg))
    rng = random.Random(15)
    out = {"digest": pl.digest(), "samples": []}
    for pi in (0, 22):
        spec = pl.primes[pi]
        p = spec.p
        table = ref.TwiddleTable(spec)
        w = [table.root_of_length(n) for n in pl.shape]
        nodes = [tuple(rng.randrange(n) for n in pl.shape) for _ in range(n_nodes)]
        nodes[0] = (0, 0, 0)
        nodes[1] = tuple(n - 1 for n in pl.shape)
        terms = [t.terms() for t in rm.unique_entries]
        grids = []
        for node in nodes:
            pt = [pow(wk, a, p) for wk, a in zip(w, node)]
            pw = [[pow(x, e, p) for e in range(5)] for x in pt]
            vals = []
            for tm in terms:
                s = 0
                for (i, j, l), c in tm.items():
                    s += c * pw[0][i] * pw[1][j] * pw[2][l]
                vals.append(s % p)
            grids.append(vals)
        g = [np.array([grids[n][e] for n in range(len(nodes))], dtype=np.int64) for e in range(rm.k)]
        dets = ref.det_grid(g, rm.r, spec, entry_ids=rm.entry_ids)
        out["samples"].append({"prime_index": pi, "nodes": [list(x) for x in nodes],
                               "det": [int(v) for v in dets]})
    _write("c5_det_samples.json", out)


def c3_full():
    """End-to-end C3 through the reference (about 3 minutes with 8 workers)."""
    m, cfg = workloads.c3()
    rm = _ref_matrix(m)
    t0 = time.time()
    result, timings, pl = ref.run_report(rm, _ref_cfg(cfg, workers=os.cpu_count()))
    wall = time.time() - t0
    coeffs = list(result.coeffs)
    blob = repr((tuple(result.shape), tuple(coeffs), tuple(result.axis_vars))).encode()
    nz = [i for i, c in enumerate(coeffs) if c]
    rng = random.Random(16)
    picks = sorted(rng.sample(nz, 64)) + [0, len(coeffs) - 1]
    _write("c3_result.json", {"digest": pl.digest(), "sha256": hashlib.sha256(blob).hexdigest(),
                              "nonzero": len(nz), "max_bits": max(abs(c).bit_length() for c in coeffs),
                              "samples": [[i, str(coeffs[i])] for i in picks],
                              "reference_seconds": wall, "timings": timings.as_dict(),
                              "workers": os.cpu_count()})


def acceptance_exact():
    """The reference's acceptance sweeps AC3, AC5 and AC6 replayed AS WRITTEN
    (`test_acceptance.py:89-103`, `:133-156`, `:159-187`): same generators,
    seeds, trial counts and primes.  The expected values are the reference
    library's own outputs (AC3: `run(m).terms()`, which the reference test
    asserts equals `sym_det`; AC5: `det_mod`; AC6: the integers themselves,
    asserted to round-trip through `combine_tensor`)."""
    import math
    from oracles import laplace_det_mod
    out = {"ac3": [], "ac5": [], "ac6": []}
    rng = random.Random(20250808)
    for trial in range(200):
        r = rng.randint(1, 5)
        vn = rng.randint(1, 3)
        max_terms = 4 if r * vn >= 12 else 6
        rows = random_matrix_terms(rng, r, vn, 4, 100, max_terms)
        m = ref.poly_matrix(rows, tuple(f"v{i}" for i in range(vn)))
        got = ref.run(m)
        out["ac3"].append({"trial": trial, "input": m.to_dict(), "shape": list(got.shape),
                           "terms": _terms_json(got.terms())})
    rng = random.Random(5)
    specs = [ref.find_fourier_primes(1, 1, start=5, min_count=1)[0],
             ref.find_fourier_primes(4, 1, start=97, min_count=1)[0],
             ref.PrimeSpec(2013265921, 15, 27, ref.find_root_of_order(2013265921, 1 << 27)),
             ref.PrimeSpec(1811939329, 27, 26, ref.find_root_of_order(1811939329, 1 << 26))]
    for trial in range(520):
        spec = specs[trial % len(specs)]
        r = rng.randint(1, 6)
        rows = [[rng.randrange(spec.p) for _ in range(r)] for _ in range(r)]
        if trial % 3 == 0:
            for _ in range(r):
                rows[rng.randrange(r)][rng.randrange(r)] = 0
            rows[rng.randrange(r)][0] = 0
        if trial % 7 == 0 and r >= 2:
            rows[1] = rows[0][:]
        want = ref.det_mod(ref.ModMatrix.from_rows(rows, spec))
        assert want == laplace_det_mod(rows, spec.p)
        out["ac5"].append({"prime": [spec.p, spec.c, spec.q, spec.omega], "rows": rows, "det": int(want)})
    rng = random.Random(6)
    pool = [3, 5, 7, 11, 97, 65537, 1000000007, 1000000009, 2013265921, 1811939329]
    for _ in range(25):
        primes = rng.sample(pool, rng.randint(2, 6))
        product = math.prod(primes)
        values = [rng.randint(-(product - 1) // 2, product // 2) for _ in range(40)]
        specs = []
        for p in primes:
            q = (p - 1) & -(p - 1)
            specs.append([p, (p - 1) // q, q.bit_length() - 1, ref.find_root_of_order(p, q)])
        tensors = [ref.reduce_mod(ref.CoeffTensor((40,), tuple(values), ("x",)), ref.PrimeSpec(*s)) for s in specs]
        assert list(ref.combine_tensor(tensors).coeffs) == values
        out["ac6"].append({"primes": specs, "values": [str(v) for v in values],
                           "residues": [[int(v) for v in t.residues] for t in tensors]})
    _write("acceptance.json", out)


C4_RUNGS = {
    # name: (builder args, keep all terms in the fixture?)
    "C4_4src_T5T11": ((4, (5, 11), False), True),
    "C4_4src_T5T11_m": ((4, (5, 11), True), False),     # "c4a": 128^3, 10 primes
    "C4_5src_T7T11": ((5, (7, 11), False), False),      # "c4b": 128^3, 16 primes
    "C4_5src_T5T7_m": ((5, (5, 7), True), False),       # 64^4, 7 primes (largest rung)
    "C2w": (None, True),                                # C2 with coefficients U[-2^31, 2^31]
}


def _result_fixture(name, m, cfg, keep_terms):
    rm = _ref_matrix(m)
    t0 = time.time()
    result, timings, pl = ref.run_report(rm, _ref_cfg(cfg, workers=os.cpu_count()))
    wall = time.time() - t0
    coeffs = list(result.coeffs)
    blob = repr((tuple(result.shape), tuple(coeffs), tuple(result.axis_vars))).encode()
    nz = [i for i, c in enumerate(coeffs) if c]
    rng = random.Random(16)
    picks = sorted(rng.sample(nz, min(64, len(nz)))) + [0, len(coeffs) - 1]
    rec = {"name": name, "digest": pl.digest(), "input_digest": ref.workspace.digest_of(rm.to_dict()),
           "shape": list(result.shape), "primes": len(pl.primes), "r": rm.r, "k": rm.k,
           "sha256": hashlib.sha256(blob).hexdigest(), "nonzero": len(nz),
           "max_bits": max(abs(c).bit_length() for c in coeffs),
           "samples": [[i, str(coeffs[i])] for i in picks],
           "reference_seconds": wall, "timings": timings.as_dict(), "workers": os.cpu_count()}
    if keep_terms:
        rec["terms"] = _terms_json(result.terms())
    print(name, "reference run", round(wall, 1), "s", flush=True)
    return rec


def c4_full(names=None):
    """The C4 ladder (and C2-wide) end to end through the reference with all host
    cores; one fixture per rung so that a partially finished ladder is still kept."""
    path = HERE / "c4_results.json"
    have = json.loads(path.read_text()) if path.exists() else {}
    for name, (args, keep) in C4_RUNGS.items():
        if names and name not in names:
            continue
        if name in have:
            continue
        m, cfg = workloads.c2(True) if args is None else workloads.harmonic(*args)
        have[name] = _result_fixture(name, m, cfg, keep)
        _write("c4_results.json", have)


def format_cases():
    """The reference's canonical text (parsing.py:211-225) of every pinned run
    result, of the reference test forms, and of random term sets with big,
    negative, unit and zero coefficients and negative/zero exponents."""
    from polydet.parsing import format_polynomial as ref_format

    runs = json.loads((HERE / "runs.json").read_text())
    cases = []
    for run in runs:
        names = tuple(run["input"]["variables"])
        terms = {tuple(e): int(c) for e, c in run["terms"]}
        cases.append({"name": run["name"], "variables": list(names), "terms": _terms_json(terms),
                      "text": ref_format(terms, names)})
    rng = random.Random(211)
    for n in range(40):
        k = rng.randint(0, 4)
        names = tuple("abcdxyz"[:k])
        terms = {}
        for _ in range(rng.randint(0, 60)):
            e = tuple(rng.choice([0, 0, 1, 1, 2, 3, 7, 12, -1]) for _ in range(k))
            c = rng.choice([0, 1, -1, rng.randint(-10**6, 10**6), rng.randint(-2**600, 2**600),
                            rng.randint(-2**64, 2**64)])
            terms[e] = c
        cases.append({"name": "random_%d" % n, "variables": list(names), "terms": _terms_json(terms),
                      "text": ref_format(terms, names)})
    _write("format.json", cases)


def condense_cases():
    """The reference's full pivot trail (determinant.py:57-84): every record's
    step, pivot value, column and sign flag, plus the determinant."""
    rng = random.Random(57)
    cases = []
    for spec in _spec_list():
        p = spec.p
        for r in (1, 2, 3, 4, 5, 6, 8, 9, 12, 16):
            for kind in ("dense", "sparse", "permuted", "singular"):
                if kind == "dense":
                    rows = [[rng.randrange(p) for _ in range(r)] for _ in range(r)]
                elif kind == "sparse":
                    rows = [[rng.randrange(p) if rng.random() < 0.35 else 0 for _ in range(r)] for _ in range(r)]
                elif kind == "permuted":
                    perm = list(range(r))
                    rng.shuffle(perm)
                    rows = [[rng.randrange(1, p) if j == perm[i] else (rng.randrange(p) if j > perm[i] else 0)
                             for j in range(r)] for i in range(r)]
                else:
                    rows = [[rng.randrange(p) for _ in range(r)] for _ in range(r)]
                    if r > 1:
                        rows[r - 1] = list(rows[0])
                value, records = ref.condense(ref.ModMatrix.from_rows(rows, spec))
                cases.append({"prime": [spec.p, spec.c, spec.q, spec.omega], "rows": rows, "det": int(value),
                              "records": [[rec.step, int(rec.value), rec.column, bool(rec.flips_sign)]
                                          for rec in records], "note": "%s r=%d" % (kind, r)})
    _write("condense.json", cases)


if __name__ == "__main__":
    if "--condense" in sys.argv:
        condense_cases()
        sys.exit(0)
    if "--format" in sys.argv:
        format_cases()
        sys.exit(0)
    if "--acceptance" in sys.argv:
        acceptance_exact()
        sys.exit(0)
    if "--c4" in sys.argv:
        c4_full([a for a in sys.argv[2:] if not a.startswith("--")] or None)
        sys.exit(0)
    plans()
    primes()
    wide_cases()
    ntt_cases()
    det_cases()
    crt_cases()
    run_cases()
    workspace_case()
    c5_det_samples()
    if "--c3" in sys.argv:
        c3_full()
