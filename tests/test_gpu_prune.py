"""Pruned node sets (csrc/expand.cu): determinants are computed only at the
nodes {u + (N/8) v : u < U} the degree bound needs, and the rest of the grid
is extended exactly.  The resulting determinant grid -- hence every residue,
artifact and coefficient -- must equal the full grid the reference computes
(pipeline.py:374-392) bit for bit."""

import random

import numpy as np
import pytest

from paper_2010_12117_b200 import PipelineConfig, executor, native, plan, poly_matrix, run, run_report, workloads
from paper_2010_12117_b200.planner import degree_bound

pytestmark = pytest.mark.gpu


def _dense(r, vn, degs, seed, lo=-50, hi=50):
    rng = random.Random(seed)
    import itertools
    mons = list(itertools.product(*(range(d + 1) for d in degs)))

    def entry():
        return {e: rng.randint(lo, hi) for e in mons if rng.random() < 0.8}

    rows = [[entry() for _ in range(r)] for _ in range(r)]
    return poly_matrix(rows, tuple("xyzw"[:vn]))


def _grids(m, mode, prune, primes=(0,)):
    """Full determinant grid per prime from PrimeStages with pruning on/off."""
    old = executor.PRUNE
    executor.PRUNE = prune
    try:
        pl = plan(m)
        st = executor.PrimeStages(m, pl, staged=(mode == "staged"))
        out = []
        for pi in primes:
            st.forward(pi)
            st.determinants(pi)
            out.append(st.det.cpu().numpy().copy())
        return out, st.dp
    finally:
        executor.PRUNE = old


CASES = [
    # r, vn, per-variable entry degrees, seed: det degree bounds r*d give N >= 16 with 8U < N
    (10, 1, (4,), 1),          # D = 40: N 64, U 6
    (10, 2, (4, 4), 2),        # 64 x 64, both axes pruned
    (6, 2, (1, 5), 3),         # D = (6, 30): N (8, 32) -> first axis whole, second U 4 = whole
    (9, 2, (2, 5), 4),         # D = (18, 45): N (32, 64), U (3, 6)
    (10, 3, (2, 4, 3), 5),     # D = (20, 40, 30): N (32, 64, 32)
    (12, 4, (1, 2, 1, 2), 6),  # D = (12, 24, 12, 24): N (16, 32, 16, 32), 4 axes
    (40, 1, (4,), 7),          # order 40 (the benchmark kernel), D = 160: N 256, U 21/22
    (17, 2, (3, 2), 8),        # odd order, runtime-order kernel
]


@pytest.mark.parametrize("mode", ["staged", "fused"])
@pytest.mark.parametrize("r,vn,degs,seed", CASES)
def test_pruned_grid_equals_full_grid(cuda, r, vn, degs, seed, mode):
    m = _dense(r, vn, degs, seed)
    full, dp_full = _grids(m, mode, False, primes=(0, 1))
    pruned, dp = _grids(m, mode, True, primes=(0, 1))
    assert dp_full.nmap is None
    for a, b in zip(full, pruned):
        assert np.array_equal(a, b)
    # the pruning actually happened where the degree bound allows it
    D = degree_bound(m)
    want = executor.kept_u(dp.shape, D)
    assert dp.kept_u == want
    if any(want):
        assert dp.sel < dp.nodes


def test_c5_node_set():
    """C5 (D = 160 per variable on 256-node axes): 168^3 of the 256^3 nodes
    get a determinant (28.3 %; the fused kernel's u-pairs straddle rows, so the
    last axis needs no rounding to an even U); test_gpu_parity's
    test_c5_determinants_at_sampled_nodes checks computed and extended nodes
    against the reference's determinants."""
    m, cfg = workloads.c5()
    pl = plan(m, cfg)
    assert executor.kept_u(pl.shape, degree_bound(m)) == [21, 21, 21]
    assert native.node_map_size(native.node_map(pl.shape, [21, 21, 21])) == 168 ** 3


@pytest.mark.parametrize("mode", ["staged", "fused"])
def test_pruned_run_equals_unpruned_run(cuda, mode, monkeypatch):
    """Whole runs with and without pruning return the identical polynomial
    (the smallest harmonic rung: 64 x 64 grid, r = 10)."""
    m, cfg = workloads.harmonic(3, (5, 7), True)
    monkeypatch.setattr(executor, "FORCE_MODE", mode)
    monkeypatch.setattr(executor, "PRUNE", False)
    want = run(m, cfg)
    monkeypatch.setattr(executor, "PRUNE", True)
    got, timings, pl = run_report(m, cfg)
    assert got.coeffs == want.coeffs and got.shape == want.shape


def test_pruned_workspace_det_artifact_is_the_full_grid(cuda, tmp_path, monkeypatch):
    """Staged workspaces store p{i}/det: with pruning it is still the full grid,
    byte-identical to the unpruned run's artifact."""
    import hashlib
    m = _dense(10, 2, (4, 4), 2)
    files = {}
    for prune in (False, True):
        monkeypatch.setattr(executor, "PRUNE", prune)
        ws = tmp_path / ("ws%d" % prune)
        run(m, PipelineConfig(), workspace=ws)
        files[prune] = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(ws.iterdir())}
    assert files[False] == files[True]


def test_node_map_validation(cuda):
    assert native.node_map((64, 64), (0, 0)) is None
    m = native.node_map((64, 32), (6, 3))
    assert native.node_map_size(m) == 48 * 24
    with pytest.raises(ValueError):
        native.node_map_size(native.node_map((64, 8), (6, 1)))     # axis shorter than 16
    with pytest.raises(ValueError):
        native.node_map_size(native.node_map((64, 32), (8, 3)))    # 8 U = N
    with pytest.raises(ValueError):
        native.node_map_size(native.node_map((48, 32), (2, 3)))    # not a power of two


@pytest.mark.parametrize("prune", [False, True])
@pytest.mark.parametrize("r,vn,degs,seed", [(10, 2, (4, 4), 2), (40, 2, (2, 2), 7), (10, 3, (2, 4, 3), 5)])
def test_fused_multi_launch_equals_staged(cuda, monkeypatch, prune, r, vn, degs, seed):
    """The fused determinant runs in chunks of whole last-axis rows; with a tiny
    chunk every launch starts mid-grid (the per-launch row offset, the pruned
    row table).  Its grid must equal the staged computation's."""
    m = _dense(r, vn, degs, seed)
    staged, _ = _grids(m, "staged", False, primes=(0,))
    monkeypatch.setattr(executor, "FUSED_CHUNK", 512)
    fused, dp = _grids(m, "fused", prune, primes=(0,))
    assert dp.sel // executor.det_chunk_size(dp) >= 2
    assert np.array_equal(staged[0], fused[0])


@pytest.mark.parametrize("r,vn,degs,seed", [c for c in CASES if c[1] >= 1])
def test_direct_interpolation_equals_inverse_of_full_grid(cuda, r, vn, degs, seed):
    """Fused runs with every axis pruned interpolate the coefficients straight
    from the kept nodes (pdb_grid_interpolate_u32).  The residue tensor must
    equal the inverse NTT of the full (extended) determinant grid -- the
    reference's _ifft_stage output (pipeline.py:395-404) -- everywhere,
    including the zeros outside the coefficient box."""
    m = _dense(r, vn, degs, seed)
    pl = plan(m)
    st = executor.PrimeStages(m, pl, staged=False)
    if not st.dp.direct:
        pytest.skip("not every axis is pruned: kept_u %s" % (st.dp.kept_u,))
    for pi in (0, 1):
        st.forward(pi)
        st.det_kernels(pi)
        saved = st.compact.clone()
        st.interpolate_direct(pi)
        direct = st.det.cpu().numpy().copy()
        st.compact.copy_(saved)
        st.expand(pi)
        st.interpolate(pi)
        want = st.det.cpu().numpy().copy()
        assert np.array_equal(direct, want)


@pytest.mark.parametrize("r,vn,degs,seed", [(10, 2, (4, 4), 2), (10, 1, (4,), 1), (10, 3, (2, 4, 3), 5)])
def test_direct_run_equals_extended_run(cuda, monkeypatch, r, vn, degs, seed):
    m = _dense(r, vn, degs, seed)
    monkeypatch.setattr(executor, "FORCE_MODE", "fused")
    monkeypatch.setattr(executor, "DIRECT", False)
    want = run(m)
    monkeypatch.setattr(executor, "DIRECT", True)
    got = run(m)
    assert got.coeffs == want.coeffs and got.shape == want.shape


def test_kernel_timing_hook(cuda):
    """pdb_kernel_timing brackets every det_gj launch with events on its stream
    (bench.py's roofline): one record per launch, positive device time."""
    m = _dense(10, 2, (4, 4), 2)
    pl = plan(m)
    st = executor.PrimeStages(m, pl, staged=False)
    st.forward(0)
    native.kernel_timing(True)
    try:
        st.det_kernels(0)
        st.det_kernels(0)
        ms, launches = native.kernel_timing_read()
    finally:
        native.kernel_timing(False)
    per_call = -(-st.dp.sel // st.chunk)
    assert launches == 2 * per_call
    assert ms > 0
    native.kernel_timing(True)
    assert native.kernel_timing_read() == (0.0, 0)
    native.kernel_timing(False)
