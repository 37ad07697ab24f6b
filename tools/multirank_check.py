"""Sharded execution on one box: launch with torchrun (N ranks); every rank runs
the same polynomial determinant through the public API with the primes (and,
for P mod N, the grid slabs) split across ranks, and rank 0 compares the
result with a single-process run.  With one GPU, let the ranks share it:

    PDB_BENCH_DEVICE=0 PDB_DIST_BACKEND=gloo torchrun --nproc-per-node 2 \
        --master-addr 127.0.0.1 tools/multirank_check.py [c3|c4a|c1]
"""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2010_12117_b200 import run, workloads  # noqa: E402


def digest(res):
    return hashlib.sha256(repr(sorted(res.terms().items())).encode()).hexdigest()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    m, cfg = {"c3": workloads.c3, "c1": workloads.c1, "c2w": lambda: workloads.c2(True),
              "c4a": lambda: workloads.harmonic(4, (5, 11), True),
              "c4_4d": lambda: workloads.harmonic(5, (5, 7), True)}[name]()
    dev = int(os.environ.get("PDB_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    single = digest(run(m, cfg))          # before the process group exists: one-process run
    backend = os.environ.get("PDB_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    sharded = digest(run(m, cfg))
    rank, size = dist.get_rank(), dist.get_world_size()
    ok = torch.tensor([1 if sharded == single else 0], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print({"config": name, "ranks": size, "primes": None, "single": single[:16], "sharded": sharded[:16],
               "all_ranks_equal_single": bool(ok.item())})
    dist.destroy_process_group()
    if not ok.item():
        sys.exit(1)


if __name__ == "__main__":
    main()
