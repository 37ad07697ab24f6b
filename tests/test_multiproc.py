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
