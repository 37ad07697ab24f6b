"""The sharded executor on the GPU: two and three torchrun ranks share the one
B200 (gloo carries the all-gathers), each runs config C3 (22 primes: whole
rounds prime-sharded, the remainder slab-sharded) and C1 (one prime: slab-
sharded only) through the public API; every rank must return exactly the
single-process polynomial (tools/multirank_check.py)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("config,ranks", [("c1", 2), ("c3", 2), ("c3", 3)])
def test_sharded_run_equals_single_process(cuda, config, ranks):
    env = dict(os.environ, PDB_BENCH_DEVICE="0", PDB_DIST_BACKEND="gloo")
    port = str(29650 + ranks + (10 if config == "c3" else 0))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", port, str(ROOT / "tools" / "multirank_check.py"), config]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "'all_ranks_equal_single': True" in out.stdout
