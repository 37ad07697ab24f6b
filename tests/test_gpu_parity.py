"""Device parity: every kernel result equals the reference's (golden vectors
from the reference itself) or the CPU oracle's, bit for bit.  Runs on a B200
(`pytest -m gpu`)."""

import hashlib
import random

import numpy as np
import pytest

from helpers import golden
import naive
from oracle import polydet_oracle as O
from paper_2010_12117_b200 import (
    CoeffTensor,
    ModMatrix,
    ModTensor,
    PipelineConfig,
    PolyMatrix,
    PrimeSpec,
    TwiddleTable,
    combine_tensor,
    condense,
    det_grid,
    det_mod,
    executor,
    find_fourier_primes,
    mrc_digits,
    build_basis,
    ntt_forward_1d,
    ntt_forward_multi,
    ntt_inverse_1d,
    ntt_inverse_multi,
    plan,
    poly_matrix,
    run,
    run_report,
)
from paper_2010_12117_b200 import workloads

pytestmark = pytest.mark.gpu
U32 = 2**31


def _spec(quad):
    return PrimeSpec(*quad)


def test_ntt_matches_reference_golden(cuda):
    checked = 0
    for case in golden("ntt.json"):
        spec = _spec(case["prime"])
        if spec.p >= U32:
            continue
        shape = tuple(case["shape"])
        names = tuple("v%d" % i for i in range(len(shape)))
        t = ModTensor(shape, np.array(case["input"], dtype=np.int64), spec, names)
        table = TwiddleTable(spec)
        assert ntt_forward_multi(t, table).residues.tolist() == case["forward"], (spec.p, shape)
        assert ntt_inverse_multi(t, table).residues.tolist() == case["inverse"], (spec.p, shape)
        checked += 1
    assert checked > 50


def test_ntt_long_axes_global_path(cuda):
    spec = find_fourier_primes(16, 1, start=10**9, min_count=1)[0]
    rng = np.random.default_rng(1)
    for n in (16384, 65536):
        x = rng.integers(0, spec.p, n)
        fwd = ntt_forward_1d(x.tolist(), TwiddleTable(spec))
        assert fwd.tolist() == O.ntt_multi(x, (n,), spec.p, spec.omega, spec.q).tolist()
        assert ntt_inverse_1d(fwd.tolist(), TwiddleTable(spec)).tolist() == x.tolist()
    x = rng.integers(0, spec.p, 2 * 16384)
    t = ModTensor((2, 16384), x, spec, ("a", "b"))
    got = ntt_forward_multi(t, TwiddleTable(spec)).residues
    assert got.tolist() == O.ntt_multi(x, (2, 16384), spec.p, spec.omega, spec.q).tolist()


@pytest.mark.parametrize("shape", [(16,), (64, 32), (16, 8, 256), (256, 4, 2)])
def test_ntt_sparse_axes_equal_dense(cuda, shape):
    """Forward passes over axes whose input is nonzero only on the first E <= 8
    rows take the evaluation kernel; it must equal the full transform."""
    import torch
    from paper_2010_12117_b200 import native
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    ctx = native.prime_context(spec)
    rng = np.random.default_rng(len(shape))
    for E in range(1, 9):
        ext = [min(E + a, n) for a, n in enumerate(shape)]
        x = np.zeros(shape, dtype=np.int64)
        box = tuple(slice(0, e) for e in ext)
        x[box] = rng.integers(0, spec.p, [e for e in ext])
        batch = 3
        data = torch.tensor(np.concatenate([x.ravel()] * batch), dtype=torch.int64).to(torch.int32).cuda()
        ref = data.clone()
        native.ntt_multi(ctx, data, batch, shape, ext, range(len(shape)), False)
        native.ntt_multi(ctx, ref, batch, shape, None, range(len(shape)), False)
        assert torch.equal(data, ref), (shape, E)
        want = O.ntt_multi(x.ravel(), shape, spec.p, spec.omega, spec.q)
        assert data[: x.size].cpu().numpy().astype(np.int64).tolist() == want.tolist()


def test_ntt_small_naive_and_errors(cuda):
    spec = find_fourier_primes(10, 1, start=10**6, min_count=1)[0]
    table = TwiddleTable(spec)
    rng = random.Random(2)
    for n in (1, 2, 4, 8, 32):
        data = [rng.randrange(spec.p) for _ in range(n)]
        w = table.root_of_length(n)
        assert ntt_forward_1d(data, table).tolist() == naive.dft(data, w, spec.p)
        assert ntt_inverse_1d(data, table).tolist() == naive.idft(data, w, spec.p)
    with pytest.raises(ValueError, match="unsupported length"):
        ntt_forward_1d([1, 2, 3], table)
    with pytest.raises(ValueError, match="unsupported length"):
        ntt_forward_1d([0] * 2048, table)


def test_det_matches_reference_golden(cuda):
    n = 0
    for case in golden("det.json"):
        spec = _spec(case["prime"])
        if spec.p >= U32:
            continue
        grids = [np.array(g, dtype=np.int64) for g in case["grids"]]
        out = det_grid(grids, case["r"], spec, entry_ids=case["entry_ids"])
        assert out.tolist() == case["expected"], case["note"]
        n += 1
    assert n > 40


@pytest.mark.parametrize("r", [4, 9, 10, 12, 14, 15, 16, 17, 23, 24, 25, 32, 33, 40, 48, 56, 63, 64, 65, 72, 96, 128])
def test_det_random_vs_oracle_with_zero_pivots(cuda, r):
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    rng = np.random.default_rng(r)
    nodes = 700 if r <= 16 else (150 if r <= 64 else 40)
    mats = rng.integers(0, spec.p, (nodes, r, r))
    mats[::7, 0, 0] = 0                          # zero leading pivot
    mats[3::11, r // 2, :] = 0                   # singular
    mats[5::13, r - 1] = mats[5::13, 0]          # duplicate rows
    mats[6::17, :, :] = np.triu(mats[6::17, :, :])[:, ::-1, :]  # permuted structure
    grids = [mats[:, e // r, e % r] for e in range(r * r)]
    got = det_grid(grids, r, spec)
    assert got.tolist() == O.det_grid(grids, r, spec.p).tolist()


@pytest.mark.parametrize("p", [2, 3, 5, 97, 65537, 1073741789, 1073741827])
def test_det_tiny_and_small_primes(cuda, p):
    """Even p has no Montgomery form: such primes take the robust kernel; odd
    small primes exercise zero pivots on the fast paths constantly;
    1073741789 (largest prime < 2^30) is the worst case of the fast kernels'
    accumulator bounds, 1073741827 (> 2^30) takes the robust path."""
    spec = PrimeSpec(p, p - 1, 0, 1)
    rng = np.random.default_rng(p % 1000)
    for r in (3, 8, 10, 24, 40, 70):
        mats = rng.integers(0, p, (300, r, r))
        grids = [mats[:, e // r, e % r] for e in range(r * r)]
        assert det_grid(grids, r, spec).tolist() == O.det_grid(grids, r, p).tolist(), (p, r)


def test_det_dedup_ids_and_31bit_prime(cuda):
    spec = find_fourier_primes(27, 1, start=2 * 10**9, min_count=1)[0]   # 2013265921 > 2^30
    rng = np.random.default_rng(3)
    a, b = rng.integers(0, spec.p, 64), rng.integers(0, spec.p, 64)
    out = det_grid([a, b], 2, spec, entry_ids=[0, 1, 1, 0])
    assert out.tolist() == ((a * a - b * b) % spec.p).tolist()
    for r in (5, 12, 20):
        mats = rng.integers(0, spec.p, (40, r, r))
        grids = [mats[:, e // r, e % r] for e in range(r * r)]
        assert det_grid(grids, r, spec).tolist() == O.det_grid(grids, r, spec.p).tolist()


def test_condense_pivot_trail(cuda):
    spec = find_fourier_primes(4, 1, start=97, min_count=1)[0]
    rows = [[0, 0, 2], [0, 3, 1], [4, 1, 5]]
    value, records = condense(ModMatrix.from_rows(rows, spec))
    assert value == naive.cofactor_det(rows, 97)
    assert [rec.column for rec in records] == [2, 1, 0]
    assert sum(rec.flips_sign for rec in records) % 2 == 1
    value, records = condense(ModMatrix.from_rows([[0, 0], [3, 4]], spec))
    assert value == 0 and records == []
    rng = random.Random(4)
    for _ in range(20):
        r = rng.randint(1, 6)
        rows = [[rng.randrange(97) if rng.random() > 0.3 else 0 for _ in range(r)] for _ in range(r)]
        assert det_mod(ModMatrix.from_rows(rows, spec)) == naive.cofactor_det(rows, 97)


def test_condense_matches_reference_trail(cuda):
    """The full pivot trail -- every pivot value, column and sign flag -- and the
    determinant equal the reference's condensation (golden condense.json: dense,
    sparse, permuted and singular matrices, r = 1..16, seven primes incl. 97,
    2^30 < p < 2^31 and a 31-bit prime on the wide path)."""
    n = 0
    for case in golden("condense.json"):
        spec = _spec(case["prime"])
        value, records = condense(ModMatrix.from_rows(case["rows"], spec))
        assert value == case["det"], case["note"]
        assert [[rec.step, rec.value, rec.column, rec.flips_sign] for rec in records] == case["records"], case["note"]
        n += 1
    assert n == 280


def test_crt_matches_reference_golden(cuda):
    for case in golden("crt.json"):
        specs = [find_fourier_primes(6, 1, start=p, min_count=1)[0] for p in case["primes"]]
        n = len(case["residues"][0])
        tensors = [ModTensor((n,), np.array(r, dtype=np.int64), s, ("x",))
                   for r, s in zip(case["residues"], specs)]
        out = combine_tensor(tensors)
        assert [str(v) for v in out.coeffs] == case["expected"]
    basis = build_basis([3, 5, 7])
    assert mrc_digits([2, 3, 2], basis) == [2, 2, 1]


def _run_case(case):
    m = PolyMatrix.from_dict(case["input"])
    cfg = PipelineConfig(**case["config"])
    result, _, pl = run_report(m, cfg)
    assert pl.digest() == case["digest"]
    assert list(result.shape) == case["shape"]
    return result.terms(), {tuple(e): c for e, c in case["terms"]}


def test_end_to_end_matches_reference_runs(cuda):
    for case in golden("runs.json"):
        if case["config"].get("prime_start", 10**9) >= U32:
            continue
        got, want = _run_case(case)
        assert got == want, case["name"]


@pytest.mark.parametrize("mode", ["staged", "fused"])
def test_modes_agree_on_harmonic_rung(cuda, mode, monkeypatch):
    monkeypatch.setattr(executor, "FORCE_MODE", mode)
    case = next(c for c in golden("runs.json") if c["name"] == "C4_3src_T5T7_m")
    got, want = _run_case(case)
    assert got == want


@pytest.mark.parametrize("r,vn,degs,seed", [
    (3, 2, (2, 11), 1),    # r <= 8 (register kernel) on the fused layout, E = 12 > 8: Horner fill
    (9, 2, (3, 4), 2),     # padded order (RP = 16), DFT-8 fill, non-dense positions
    (10, 3, (1, 1, 6), 3), # 3 variables, E = 7
    (10, 2, (1, 2), 4),    # short last axis (N = 32): U-group divisibility edge
    (16, 2, (1, 2), 6),    # compile-time order 16, dense DFT-8 fill
    (34, 1, (1,), 5),      # compile-time order 40 with 6 padded rows, one variable
])
def test_fused_mode_edge_shapes_vs_oracle(cuda, monkeypatch, r, vn, degs, seed):
    """The fused path (partial forward NTT + in-kernel last-axis evaluation) at
    shapes that select each fill variant, against the oracle pipeline."""
    import itertools
    rng = random.Random(seed)
    names = ("x", "y", "z")[:vn]

    def entry():
        mons = list(itertools.product(*(range(d + 1) for d in degs)))
        return {e: rng.randint(-50, 50) for e in rng.sample(mons, min(len(mons), 6))}

    rows = [[entry() for _ in range(r)] for _ in range(r)]
    m = poly_matrix(rows, names)
    monkeypatch.setattr(executor, "FORCE_MODE", "fused")
    pl = plan(m)
    got = run(m)
    want, _ = O.run_pipeline([t.terms() for t in m.unique_entries], m.entry_ids, m.r, pl.shape,
                             [(s.p, s.omega, s.q) for s in pl.primes])
    assert list(got.coeffs) == want


def test_workspace_artifacts_byte_identical_to_reference(cuda, tmp_path):
    g = golden("workspace.json")
    m = PolyMatrix.from_dict(g["input"])
    units = []
    run(m, PipelineConfig(progress=units.append), workspace=tmp_path / "ws")
    assert units == g["units"]
    files = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in (tmp_path / "ws").iterdir()}
    assert files == g["files"]
    assert (tmp_path / "ws" / "manifest").read_text().splitlines() == g["manifest"]


class _Abort(Exception):
    pass


def _abort_after(n):
    seen = {"k": 0}

    def hook(unit):
        seen["k"] += 1
        if seen["k"] >= n:
            raise _Abort(unit)
    return hook


def test_kill_and_resume_every_boundary(cuda, tmp_path):
    from paper_2010_12117_b200 import resume

    rng = random.Random(7)
    rows = naive.random_poly_matrix(rng, 3, 2, 3, 60, 4, dup=0.3)
    m = poly_matrix(rows, ("x", "y"))
    units = []
    reference = run(m, PipelineConfig(progress=units.append))
    assert reference.terms() == naive.symbolic_det(rows, 2)
    pl = plan(m)
    assert len(units) == pl.prime_count * (m.k + 2) + 1
    for cut in range(1, len(units)):
        ws = tmp_path / ("ws%d" % cut)
        with pytest.raises(_Abort):
            run(m, PipelineConfig(progress=_abort_after(cut)), workspace=ws)
        seen = []
        resumed = resume(ws, PipelineConfig(progress=seen.append))
        assert resumed.coeffs == reference.coeffs
        assert len(seen) == len(units) - cut
    again = []
    assert run(m, PipelineConfig(progress=again.append), workspace=tmp_path / "ws1").coeffs == reference.coeffs
    assert again == []


def test_edge_cases(cuda):
    assert run(poly_matrix([[{(1,): 1}]], ("x",))).terms() == {(1,): 1}
    assert run(poly_matrix([[{}, {}], [{}, {}]], ("x",))).terms() == {}
    assert run(poly_matrix([[{(0,): 3}, {(0,): 1}], [{(0,): 4}, {(0,): 2}]], ("x",))).terms() == {(0,): 2}
    m = poly_matrix([[{(): 2}, {(): 1}], [{(): 5}, {(): 7}]], ())
    out = run(m)
    assert out.shape == () and out.terms() == {(): 9}
    m = poly_matrix([[{(1, 0): 1}, {(0, 1): 1}], [{(0, 0): 1}, {(1, 0): 1}]], ("x", "y"))
    assert run(m).terms() == {(2, 0): 1, (0, 1): -1}
    a = run(m, PipelineConfig(prime_start=10**9)).coeffs
    assert run(m, PipelineConfig(prime_start=15 * 10**8)).coeffs == a


def test_random_matrices_vs_symbolic(cuda):
    rng = random.Random(20250808)
    for _ in range(30):
        r = rng.randint(1, 5)
        vn = rng.randint(1, 3)
        rows = naive.random_poly_matrix(rng, r, vn, rng.randint(0, 3), 100, 4)
        assert run(poly_matrix(rows, "xyz"[:vn])).terms() == naive.symbolic_det(rows, vn)


def test_c3_end_to_end_matches_reference(cuda):
    g = golden("c3_result.json")
    m, cfg = workloads.c3()
    result, timings, pl = run_report(m, cfg)
    assert pl.digest() == g["digest"]
    coeffs = result.coeffs
    for idx, val in g["samples"]:
        assert coeffs[idx] == int(val)
    blob = repr((tuple(result.shape), tuple(coeffs), tuple(result.axis_vars))).encode()
    assert hashlib.sha256(blob).hexdigest() == g["sha256"]


@pytest.mark.parametrize("mode", ["fused", "staged"])
def test_c5_determinants_at_sampled_nodes(cuda, mode):
    g = golden("c5_det_samples.json")
    m, cfg = workloads.c5()
    pl = plan(m, cfg)
    assert pl.digest() == g["digest"]
    if mode == "staged" and cuda.cuda.get_device_properties(0).total_memory < 150 << 30:
        pytest.skip("staged C5 needs ~110 GB")
    stages = executor.PrimeStages(m, pl, staged=(mode == "staged"))
    N = pl.shape
    for sample in g["samples"]:
        pi = sample["prime_index"]
        stages.forward(pi)
        stages.determinants(pi)
        det = stages.det.cpu().numpy().view(np.uint32)
        idx = [(a * N[1] + b) * N[2] + c for a, b, c in sample["nodes"]]
        assert det[idx].tolist() == sample["det"]
        # size-independent property: interpolation then evaluation is the identity
        before = stages.det.clone()
        stages.interpolate(pi)
        from paper_2010_12117_b200 import native
        native.ntt_multi(stages.ctx(pi), stages.det, 1, N, None, range(3), False)
        assert cuda.equal(before, stages.det)
    del stages


@pytest.mark.parametrize("config,seed", [("c3", 9), ("c5", 10)])
def test_schwartz_zippel_full_size(cuda, config, seed):
    """Evaluate the final polynomial (C3: 117 649 terms; C5: 4.17 M terms of up to
    449 bits, 23 primes, the benchmark's fused path end to end) at a random point
    mod a fresh prime and compare with the determinant of the entry-wise
    evaluated matrix."""
    m, cfg = getattr(workloads, config)()
    out = run(m, cfg)
    q = 2**61 - 1
    rng = random.Random(seed)
    point = [rng.randrange(q) for _ in range(3)]
    lhs = naive.poly_eval(out.terms(), point, q)
    mat = [[naive.poly_eval(m.entry(i, j).terms(), point, q) for j in range(m.r)] for i in range(m.r)]
    # Gaussian elimination mod q (q prime)
    det = 1
    for c in range(m.r):
        piv = next(i for i in range(c, m.r) if mat[i][c] % q)
        if piv != c:
            mat[c], mat[piv] = mat[piv], mat[c]
            det = -det
        det = det * mat[c][c] % q
        inv = pow(mat[c][c], -1, q)
        for i in range(c + 1, m.r):
            f = mat[i][c] * inv % q
            mat[i] = [(x - f * y) % q for x, y in zip(mat[i], mat[c])]
    assert lhs == det % q


def test_predict_on_real_matrix(cuda):
    """Reference test_pipeline.py:212-229: the forecast's fields and formula."""
    from decimal import Decimal
    from fractions import Fraction
    from paper_2010_12117_b200 import predict, predicted_total
    rng = random.Random(8)
    rows = [[{(e,): rng.randint(-9, 9) for e in range(4)} for _ in range(2)] for _ in range(2)]
    m = poly_matrix(rows, ("x",))
    pl = plan(m)
    forecast = predict(m, pl, sample_size=2)
    assert forecast.prime_count == pl.prime_count and forecast.order == 2
    assert len(forecast.sample_seconds) == 2
    assert forecast.replication == Fraction(m.k, 4)
    mean = sum(forecast.sample_seconds) / 2
    assert forecast.total_seconds == predicted_total(pl.prime_count, pl.r, pl.unique_count, mean)
    assert forecast.mean_rounded == Decimal(repr(mean)).quantize(Decimal("0.01"))
    with pytest.raises(ValueError):
        predict(m, pl, 0)


def test_integration_ctypes_stub_runs(cuda):
    """The Option B ctypes stub printed in INTEGRATION.md (a maintainer's
    reference-side binding of pdb_det_batch_u32) runs as written and agrees
    with the oracle."""
    import re
    from pathlib import Path
    from paper_2010_12117_b200 import native
    text = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    block = re.search(r"## Option B.*?```python\n(.*?)```", text, re.S).group(1)
    block = block.replace('ctypes.CDLL("libpolydet_b200.so")', "ctypes.CDLL(%r)" % str(native.LIB_PATH))
    env = {}
    exec(compile(block, "INTEGRATION.md", "exec"), env)
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    rng = np.random.default_rng(11)
    grids = [rng.integers(0, spec.p, 300) for _ in range(144)]
    assert env["det_grid"](grids, 12, spec).tolist() == O.det_grid(grids, 12, spec.p).tolist()


@pytest.mark.parametrize("mode", ["staged", "fused"])
def test_many_variables_vs_oracle(cuda, monkeypatch, mode):
    """Nine variables (grid 4^9 = 262 144 nodes): NTTs over nine axes, fused
    layout with eleven dimensions."""
    rng = random.Random(99)
    nv = 9
    names = tuple("v%d" % i for i in range(nv))

    def entry():
        return {tuple(int(i == a) for i in range(nv)): rng.randint(-5, 5) for a in rng.sample(range(nv), 3)}

    rows = [[entry() for _ in range(3)] for _ in range(3)]
    m = poly_matrix(rows, names)
    monkeypatch.setattr(executor, "FORCE_MODE", mode)
    pl = plan(m)
    got = run(m)
    want, _ = O.run_pipeline([t.terms() for t in m.unique_entries], m.entry_ids, m.r, pl.shape,
                             [(s.p, s.omega, s.q) for s in pl.primes])
    assert list(got.coeffs) == want
    assert got.terms() == naive.symbolic_det(rows, nv)


def test_fused_mode_workspace_kill_and_resume(cuda, tmp_path, monkeypatch):
    """Grids too large for the staged layout checkpoint per prime (p{i}/ifft
    units only, which is all the reference's executor needs to resume); a
    run killed after any unit resumes to the same result."""
    from paper_2010_12117_b200 import resume
    monkeypatch.setattr(executor, "STAGED_LIMIT", 0)   # force the fused layout even with a workspace
    m, cfg = workloads.harmonic(3, (5, 7), True)
    reference = run(m, cfg)
    units = []
    run(m, PipelineConfig(progress=units.append), workspace=tmp_path / "full")
    pl = plan(m, cfg)
    assert units == ["p%d/ifft" % i for i in range(pl.prime_count)] + ["crt"]
    for cut in range(1, len(units)):
        ws = tmp_path / ("ws%d" % cut)
        with pytest.raises(_Abort):
            run(m, PipelineConfig(progress=_abort_after(cut)), workspace=ws)
        seen = []
        assert resume(ws, PipelineConfig(progress=seen.append)).coeffs == reference.coeffs
        assert seen == units[cut:]


def test_resume_reference_written_partial_workspace(cuda, tmp_path):
    """Cross-resume: a workspace the reference itself wrote and was killed in
    (tests/golden/make_partial_ws.py, after 7 of 17 units) is finished by this
    package, which computes exactly the remaining units and returns the
    reference's result."""
    import json
    import shutil
    from pathlib import Path
    from paper_2010_12117_b200 import resume
    here = Path(__file__).resolve().parent / "golden"
    meta = json.loads((here / "ref_partial_ws.json").read_text())
    ws = tmp_path / "ws"
    shutil.copytree(here / "ref_partial_ws", ws)
    seen = []
    got = resume(ws, PipelineConfig(progress=seen.append))
    assert seen == meta["remaining_units"]
    assert list(got.shape) == meta["shape"]
    assert got.terms() == {tuple(e): c for e, c in meta["terms"]}
    # the completed workspace reloads without recomputation
    again = []
    assert resume(ws, PipelineConfig(progress=again.append)).coeffs == got.coeffs
    assert again == []


@pytest.mark.parametrize("p", [1000000513, 1041682561, 1041682661])
@pytest.mark.parametrize("r", [33, 40])
def test_paired_pivot_blocks_at_the_accumulator_bound(cuda, r, p, monkeypatch):
    """Order-40 kernels update the trailing matrix of their first two pivot
    blocks in one pass (17 products per reduction) when p < 1.0417e9:
    1041682561 is the largest prime inside that bound (entries near p - 1 are
    the worst case), 1041682661 the smallest outside it (unpaired kernel).  Both
    equal the oracle and the unpaired kernel (PDB_GJ_NO_PAIR=1); the fused C5
    kernel is paired too (test_c5_determinants_at_sampled_nodes)."""
    spec = PrimeSpec(p, p - 1, 0, 1)
    rng = np.random.default_rng(p % 977 + r)
    mats = rng.integers(0, p, (400, r, r))
    mats[::3] = p - 1 - rng.integers(0, 3, (len(mats[::3]), r, r))   # entries at the top of the range
    mats[::11, 0, 0] = 0
    mats[5::13, 9, :] = 0                                           # singular inside the second block
    grids = [mats[:, e // r, e % r] for e in range(r * r)]
    want = O.det_grid(grids, r, p).tolist()
    assert det_grid(grids, r, spec).tolist() == want
    monkeypatch.setenv("PDB_GJ_NO_PAIR", "1")
    assert det_grid(grids, r, spec).tolist() == want


@pytest.mark.parametrize("r", [16, 24, 40])
def test_singular_leading_blocks_take_the_robust_path(cuda, r):
    """The compile-time-order kernels invert each 8x8 pivot block by 4x4 blocks
    and flag a node when a 4x4 block or its Schur complement is singular, i.e.
    when a leading principal minor of order 4k vanishes.  Matrices built with
    exactly such a minor (row t-1 restricted to the first t columns is a
    combination of the rows above it, t = 4, 8, 12, ...) but generically
    nonsingular overall go to det_robust and still equal the oracle; so do
    singular matrices and the plain random ones around them."""
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    p = spec.p
    rng = np.random.default_rng(7 + r)
    mats = []
    for t in range(4, r, 4):
        for _ in range(6):
            m = rng.integers(0, p, (r, r))
            coef = rng.integers(0, p, t - 1)
            m[t - 1, :t] = (coef[:, None] * m[: t - 1, :t] % p).sum(axis=0) % p
            mats.append(m)
    mats.append(np.zeros((r, r), dtype=np.int64))
    sing = rng.integers(0, p, (r, r))
    sing[-1] = (3 * sing[0] + 5 * sing[1]) % p
    mats.append(sing)
    mats += [rng.integers(0, p, (r, r)) for _ in range(40)]
    mats = np.stack(mats)
    grids = [mats[:, e // r, e % r] for e in range(r * r)]
    want = O.det_grid(grids, r, p).tolist()
    got = det_grid(grids, r, spec).tolist()
    assert got == want
    assert sum(1 for v in want if v) >= len(want) - 2   # only the two singular ones vanish


@pytest.mark.parametrize("r", [13, 16, 21, 24, 30, 32, 36, 40])
def test_compile_time_and_runtime_order_kernels_agree(cuda, r, monkeypatch):
    """Padded orders 16, 24, 32 and 40 run compile-time-order kernels (the staged
    16 and 40 ones with a 4-pivot tail); PDB_GJ_NO_RPC=1 selects the generic
    runtime-order kernel.  Both equal the oracle, zero pivots included."""
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    rng = np.random.default_rng(100 + r)
    mats = rng.integers(0, spec.p, (300, r, r))
    mats[::9, 0, 0] = 0
    mats[4::13, r - 2, :] = 0
    grids = [mats[:, e // r, e % r] for e in range(r * r)]
    want = O.det_grid(grids, r, spec.p).tolist()
    assert det_grid(grids, r, spec).tolist() == want
    monkeypatch.setenv("PDB_GJ_NO_RPC", "1")
    assert det_grid(grids, r, spec).tolist() == want
