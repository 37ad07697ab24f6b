"""The sharded executor on the GPU: two and three torchrun ranks share the one
B200 (gloo carries the collectives), each runs config C3 (22 primes: whole
rounds prime-sharded, the remainder slab-sharded, CRT sharded by coefficient
range), C1 (one prime: slab-sharded only), C2-wide (u64 residues) and a C4
rung through the public API; every rank must return exactly the
single-process polynomial (tools/multirank_check.py).  With two or more GPUs
visible the same check runs one rank per GPU over NCCL."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("config,ranks", [("c1", 2), ("c3", 2), ("c3", 3), ("c2w", 2), ("c4a", 3)])
def test_sharded_run_equals_single_process(cuda, config, ranks):
    env = dict(os.environ, PDB_BENCH_DEVICE="0", PDB_DIST_BACKEND="gloo")
    port = str(29650 + ranks + 10 * ["c1", "c3", "c2w", "c4a"].index(config))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", port, str(ROOT / "tools" / "multirank_check.py"), config]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "'all_ranks_equal_single': True" in out.stdout


@pytest.mark.parametrize("config", ["c3", "c1"])
def test_nccl_one_rank_per_gpu(cuda, config):
    """NCCL, one process per GPU (all_to_all of residues, all-gather of the
    compact CRT rows): needs >= 2 visible GPUs."""
    if cuda.cuda.device_count() < 2:
        pytest.skip("NCCL sharding needs >= 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("PDB_BENCH_DEVICE", "PDB_DIST_BACKEND")}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29710 + len(config)),
           str(ROOT / "tools" / "multirank_check.py"), config]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "'all_ranks_equal_single': True" in out.stdout
