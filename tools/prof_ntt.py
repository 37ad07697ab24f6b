"""Per-kernel timing of the C5 step's non-determinant stages (forward
evaluation, grid extension, inverse NTT) for profiling.

    python tools/prof_ntt.py [--reps 5] [--config c5|c3]

Prints one JSON object: milliseconds per stage (CUDA events, best of reps) and
the stage's algorithmic HBM bytes (u32 words read + written once per pass).
Run under `ncu -k regex:'ntt_axis|grid_'` for the kernel captures.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2010_12117_b200 import executor, plan, workloads  # noqa: E402


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
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--config", default="c5")
    args = ap.parse_args()
    m, cfg = workloads.c5() if args.config == "c5" else workloads.c3()
    pl = plan(m, cfg)
    st = executor.PrimeStages(m, pl, staged=False)
    st.step(0)
    nodes = pl.node_count
    out = {"config": args.config, "shape": list(pl.shape), "nodes": nodes, "kept_u": st.dp.kept_u}
    out["forward_ms"] = timed(lambda: st.forward(0), args.reps)
    out["expand_ms"] = timed(lambda: st.expand(0), args.reps)
    out["inverse_ms"] = timed(lambda: st.interpolate(0), args.reps)
    if st.dp.direct:   # coefficients straight from the kept nodes (replaces expand + inverse)
        st.det_kernels(0)
        saved = st.compact.clone()
        out["copy_ms"] = timed(lambda: st.compact.copy_(saved), args.reps)
        out["direct_ms"] = timed(lambda: (st.compact.copy_(saved), st.interpolate_direct(0)), args.reps) \
            - out["copy_ms"]
    vn = len(pl.shape)
    inv_bytes = 2 * 4 * nodes * vn
    out["inverse_algorithmic_bytes"] = inv_bytes
    out["inverse_gbs"] = inv_bytes / (out["inverse_ms"] * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
