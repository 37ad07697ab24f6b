"""Kernel-level determinant throughput (dets/s, Gupd/s) for profiling.

    python tools/det_bench.py [--r 4,16,40] [--nodes N] [--fused] [--reps 3]

Staged mode: random residue grids already in HBM (k = r^2 grids of `nodes`
u32), times pdb_det_batch_u32.  --fused: the C5 workload's first prime,
partial transform resident, times pdb_eval_det_fused_u32 over `nodes` nodes.
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2010_12117_b200 import executor, find_fourier_primes, native, plan, workloads  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", default="4,16,40")
    ap.add_argument("--nodes", type=int, default=1 << 20)
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--pruned", action="store_true", help="profile only the pruned fused launch")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    out = {}
    spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
    ctx = native.prime_context(spec)
    for r in [int(x) for x in args.r.split(",") if x]:
        n = args.nodes
        grids = torch.randint(0, spec.p, (r * r, n), dtype=torch.int64, device="cuda").to(torch.int32)
        ids = torch.arange(r * r, dtype=torch.int32, device="cuda")
        det = torch.empty(n, dtype=torch.int32, device="cuda")
        scratch = native.scratch_tensor(native.det_scratch_bytes(r, n))
        t = timed(lambda: native.det_batch(ctx, grids, n, ids, r, 0, n, det, scratch), args.reps)
        W = (r ** 3 - r) // 3
        out["staged_r%d" % r] = {"nodes": n, "s": t, "dets_per_s": n / t, "gupd_per_s": n * W / t / 1e9,
                                 "bytes_per_s": 4.0 * (r * r + 1) * n / t}
        del grids
    if args.fused or args.pruned:
        m, cfg = workloads.c5()
        pl = plan(m, cfg)
        st = executor.PrimeStages(m, pl, staged=False)
        st.forward(0)
        n = min(args.nodes, pl.node_count)
        dp = st.dp
        st.scratch = native.scratch_tensor(native.det_scratch_bytes(pl.r, max(n, st.chunk)))
        c = st.ctx(0)
        W = (40 ** 3 - 40) // 3
        if args.fused:
            t = timed(lambda: native.eval_det_fused(c, st.work, dp.outer, dp.E, dp.k, pl.shape[-1], dp.ids, pl.r, 0,
                                                    n, st.det[:n], st.scratch), args.reps)
            out["fused_c5"] = {"nodes": n, "s": t, "dets_per_s": n / t, "gupd_per_s": n * W / t / 1e9}
        if dp.nmap is not None:   # the same kernel over the kept (pruned) node set
            row = dp.klen[-1]
            npr = max(row, min(args.nodes, dp.sel) // row * row)
            t = timed(lambda: native.eval_det_fused_map(c, st.work, dp.outer, dp.E, dp.k, pl.shape[-1], dp.ids,
                                                        pl.r, dp.nmap, 0, npr, st.compact[:npr], st.scratch),
                      args.reps)
            out["fused_c5_pruned"] = {"nodes": npr, "s": t, "dets_per_s": npr / t, "gupd_per_s": npr * W / t / 1e9}
        tf = timed(lambda: st.forward(0), args.reps)
        ti = timed(lambda: st.interpolate(0), args.reps)
        out["c5_forward_s"] = tf
        out["c5_inverse_s"] = ti
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
