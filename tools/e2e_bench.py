"""End-to-end seconds per polynomial determinant through the public API
(BASELINE.json metric, second half): `run_report(m, cfg)` on one GPU for the
SURVEY.md 8(d) configurations, with the per-stage device times.

    python tools/e2e_bench.py [--configs c1,c2,c2w,c3,c4a,c4b,c5] [--reps 2]

Prints one JSON object per configuration: matrix build + plan seconds, the
wall time of run_report (best of --reps after one warm-up run), its
StageTimings (fft/det/ifft/crt device seconds), and the result's size.
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2010_12117_b200 import plan, run_report, workloads  # noqa: E402

CONFIGS = {
    "c1": lambda: workloads.c1(),
    "c2": lambda: workloads.c2(),
    "c2w": lambda: workloads.c2(wide=True),
    "c3": lambda: workloads.c3(),
    # harmonic-elimination rungs of SURVEY.md 8(d) (C4): reference 8-worker CPU times 202.1 s / 440.1 s
    "c4a": lambda: workloads.harmonic(4, (5, 11), True),
    "c4b": lambda: workloads.harmonic(5, (7, 11), False),
    "c5": lambda: workloads.c5(),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c2w,c3,c4a,c4b,c5")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    for name in args.configs.split(","):
        t0 = time.perf_counter()
        m, cfg = CONFIGS[name]()
        t1 = time.perf_counter()
        pl = plan(m, cfg)
        t2 = time.perf_counter()
        run_report(m, cfg)   # warm-up: contexts, twiddles, allocator
        best = None
        for _ in range(args.reps):
            s = time.perf_counter()
            result, timings, _ = run_report(m, cfg)
            wall = time.perf_counter() - s
            if best is None or wall < best[0]:
                best = (wall, timings, result)
        wall, timings, result = best
        nz = [c for c in result.coeffs if c]
        print(json.dumps({
            "config": name, "r": m.r, "k": m.k, "vars": len(pl.variables), "shape": list(pl.shape),
            "primes": pl.prime_count, "nodes": pl.node_count,
            "build_s": t1 - t0, "plan_s": t2 - t1, "run_report_s": wall,
            "stages_s": {"fft": timings.fft, "det": timings.det, "ifft": timings.ifft, "crt": timings.crt},
            "nonzero_terms": len(nz), "max_bits": max((abs(c).bit_length() for c in nz), default=0),
        }), flush=True)


if __name__ == "__main__":
    main()
