"""Multi-process sharding on CPU (gloo, world size 2 and 3): the prime
assignment and the residue gather reassemble exactly the single-process
residue block, so the CRT input -- and hence the result -- is identical for
any device count.  The per-prime compute here is the CPU oracle (test
infrastructure); on the GPU the same host logic wraps the device kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import golden
from oracle import polydet_oracle as O
from paper_2010_12117_b200 import PolyMatrix, plan, shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _residues(m, pl, pi):
    spec = pl.primes[pi]
    terms = [t.terms() for t in m.unique_entries]
    _, res = O.run_pipeline(terms, m.entry_ids, m.r, pl.shape, [(spec.p, spec.omega, spec.q)])
    return res[0]


def _worker(rank, size, port, case, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    m = PolyMatrix.from_dict(case["input"])
    pl = plan(m)
    mine = shard.my_primes(pl.prime_count, rank, size)
    local = torch.tensor(np.stack([_residues(m, pl, pi) for pi in mine]), dtype=torch.int64) \
        if mine else torch.zeros((0, pl.node_count), dtype=torch.int64)
    full = shard.gather_residues(local, pl.prime_count, rank, size)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_residues_match_single_process(tmp_path, size):
    case = next(c for c in golden("runs.json") if c["name"] == "C2")
    m = PolyMatrix.from_dict(case["input"])
    pl = plan(m)
    out = tmp_path / "full.npy"
    mp.spawn(_worker, args=(size, _free_port(), case, str(out)), nprocs=size, join=True)
    full = np.load(out)
    single = np.stack([_residues(m, pl, pi) for pi in range(pl.prime_count)])
    assert np.array_equal(full, single)
    coeffs = O.crt_combine(list(full), [s.p for s in pl.primes])
    want = {tuple(e): c for e, c in case["terms"]}
    got = {(i,): c for i, c in enumerate(coeffs) if c}
    assert got == want


def test_prime_assignment_balanced():
    for P in (1, 7, 22, 23, 64):
        for G in (1, 2, 4, 8):
            parts = [shard.my_primes(P, g, G) for g in range(G)]
            assert sorted(sum(parts, [])) == list(range(P))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _slab_worker(rank, size, port, case, out_path):
    """Slab-sharded primes: each rank computes the determinants of its slab of
    the slowest axis (oracle det on the oracle's entry grids), the slabs are
    all-gathered and every rank interpolates the full grid."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    m = PolyMatrix.from_dict(case["input"])
    pl = plan(m)
    whole, slab = shard.split_primes(pl.prime_count, size)
    n0 = pl.shape[0]
    inner = pl.node_count // n0
    lo, hi = shard.my_slab(n0, rank, size)
    rows = []
    for pi in slab:
        spec = pl.primes[pi]
        grids = [O.ntt_multi(O.reduce_entry(t.terms(), pl.shape, spec.p), pl.shape, spec.p, spec.omega, spec.q)
                 for t in m.unique_entries]
        part = O.det_grid([g[lo * inner: hi * inner] for g in grids], m.r, spec.p, m.entry_ids)
        full = shard.gather_slabs(torch.tensor(np.asarray(part, dtype=np.int64)), n0, inner, rank, size)
        rows.append(O.ntt_multi(full.numpy(), pl.shape, spec.p, spec.omega, spec.q, inverse=True))
    if rank == 0:
        np.save(out_path, np.stack(rows))
    dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3, 5])
def test_slab_sharded_primes_match_single_process(tmp_path, size):
    case = next(c for c in golden("runs.json") if c["name"] == "C2")
    m = PolyMatrix.from_dict(case["input"])
    pl = plan(m)
    whole, slab = shard.split_primes(pl.prime_count, size)
    assert whole + len(slab) == pl.prime_count and len(slab) == pl.prime_count % size
    out = tmp_path / "slab.npy"
    mp.spawn(_slab_worker, args=(size, _free_port(), case, str(out)), nprocs=size, join=True)
    got = np.load(out)
    assert np.array_equal(got, np.stack([_residues(m, pl, pi) for pi in slab]))


def _partial_worker(rank, size, port, case, force_rs, out_path):
    """Slab-sharded primes without a mid-pipeline exchange: each rank
    interpolates its slab of determinants alone (zero elsewhere; the inverse
    transform is linear) and the partial rows are summed by a reduce-scatter
    over the CRT's coefficient ranges."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    m = PolyMatrix.from_dict(case["input"])
    pl = plan(m)
    _, slab = shard.split_primes(pl.prime_count, size)
    n0 = pl.shape[0]
    inner = pl.node_count // n0
    lo, hi = shard.my_slab(n0, rank, size)
    rows = []
    for pi in slab:
        spec = pl.primes[pi]
        grids = [O.ntt_multi(O.reduce_entry(t.terms(), pl.shape, spec.p), pl.shape, spec.p, spec.omega, spec.q)
                 for t in m.unique_entries]
        dets = np.zeros(pl.node_count, dtype=np.int64)
        dets[lo * inner: hi * inner] = O.det_grid([g[lo * inner: hi * inner] for g in grids], m.r, spec.p,
                                                  m.entry_ids)
        rows.append(O.ntt_multi(dets, pl.shape, spec.p, spec.omega, spec.q, inverse=True))
    if force_rs:
        shard._backend = lambda: "nccl"     # exercise reduce_scatter_tensor
    part = shard.reduce_scatter_rows(torch.tensor(np.stack(rows), dtype=torch.int32),
                                     [pl.primes[pi].p for pi in slab], rank, size)
    clo, chi = shard.coefficient_range(pl.node_count, rank, size)
    single = np.stack([_residues(m, pl, pi) for pi in slab])
    ok = part.dtype == torch.int32 and np.array_equal(part.numpy().astype(np.int64), single[:, clo:chi])
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        np.save(out_path, flag.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("size,force_rs", [(2, False), (3, False), (5, False), (2, True), (3, True)])
def test_slab_partial_rows_reduce_scatter(tmp_path, size, force_rs):
    case = next(c for c in golden("runs.json") if c["name"] == "C2")
    out = tmp_path / "flag.npy"
    mp.spawn(_partial_worker, args=(size, _free_port(), case, force_rs, str(out)), nprocs=size, join=True)
    assert np.load(out).tolist() == [1]


def test_slab_partition_covers_axis():
    for n0 in (1, 3, 16, 256):
        for G in (1, 2, 3, 8):
            spans = [shard.my_slab(n0, g, G) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n0
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _exchange_worker(rank, size, port, P, n, force_a2a, out_path):
    """CRT sharding: the all-to-all of residue rows leaves each rank every
    prime's residues of its coefficient range; the compact CRT rows of all
    ranks all-gather back into ascending order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    rng = np.random.default_rng(7)
    full = torch.tensor(rng.integers(0, 2**31 - 1, (P, n)), dtype=torch.int64)
    whole = (P // size) * size
    local = full[shard.my_primes(whole, rank, size)]
    if force_a2a:
        shard._backend = lambda: "nccl"     # exercise all_to_all_single (gloo implements it on CPU)
    block = shard.exchange_residues(local, whole, rank, size)
    lo, hi = shard.coefficient_range(n, rank, size)
    ok = bool(torch.equal(block, full[:whole, lo:hi]))
    # compact rows: this rank's "nonzero" positions are those with an odd first residue
    pos = torch.nonzero(block[0] % 2 == 1).squeeze(1)
    count = int(pos.numel())
    width = 3
    limbs = torch.zeros((max(count, 1), 5), dtype=torch.int32)
    limbs[:count, 0] = (pos + lo).to(torch.int32)
    limbs[:count, 2] = rank
    neg = (pos % 3 == 0).to(torch.uint8)
    g_l, g_i, g_n = shard.gather_compact(count, limbs, pos + lo, neg, width, rank, size)
    want_pos = torch.nonzero(full[0] % 2 == 1).squeeze(1) if whole else torch.zeros(0, dtype=torch.int64)
    ok = ok and torch.equal(g_i, want_pos) and torch.equal(g_l[:, 0].to(torch.int64), want_pos)
    ok = ok and g_l.shape[1] == width and torch.equal(g_n, ((want_pos - torch.tensor(
        [shard.coefficient_range(n, g, size)[0] for g in range(size)])[
            torch.searchsorted(torch.tensor([shard.coefficient_range(n, g, size)[1] for g in range(size)]),
                               want_pos, right=True)]) % 3 == 0).to(torch.uint8))
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        np.save(out_path, flag.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("size,P,n,force_a2a", [(2, 22, 1000, False), (3, 23, 1001, False), (5, 23, 64, False),
                                                (2, 22, 1000, True), (3, 9, 517, True)])
def test_crt_exchange_and_gather(tmp_path, size, P, n, force_a2a):
    out = tmp_path / "flag.npy"
    mp.spawn(_exchange_worker, args=(size, _free_port(), P, n, force_a2a, str(out)), nprocs=size, join=True)
    assert np.load(out).tolist() == [1]


def test_coefficient_ranges_cover():
    for n in (1, 7, 262144, 16777216):
        for G in (1, 2, 3, 8):
            spans = [shard.coefficient_range(n, g, G) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
