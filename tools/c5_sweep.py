"""C5 throughput sweep over the prime count on one GPU (BASELINE configs[4]:
"a throughput sweep over prime count").

    python tools/c5_sweep.py [--stage 1,2,4,8,16] [--full 23,32,64]

* P < 23 (`--stage`): the plan would be invalid for CRT, so these are
  stage-only -- forward evaluation + det at all 16.7 M nodes + inverse NTT for
  the first P primes of the C5 plan (PrimeStages.step), CUDA-event timed.
* P >= 23 (`--full`): complete runs through the public API,
  `run_report(m, PipelineConfig(min_primes=P))`, wall seconds and stage times.
  Every full run must return the same polynomial (more primes than the bound
  needs cannot change an exact result); the script checks it.
One JSON line per point.
"""
import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2010_12117_b200 import PipelineConfig, executor, plan, run_report, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", default="1,2,4,8,16")
    ap.add_argument("--full", default="23,32,64")
    args = ap.parse_args()
    m, cfg = workloads.c5()
    pl = plan(m, cfg)
    st = executor.PrimeStages(m, pl, staged=False)
    st.step(0)                       # warm-up (module load, twiddles, first launch)
    torch.cuda.synchronize()
    for P in [int(x) for x in args.stage.split(",") if x]:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(P):
            st.step(i % pl.prime_count)
        b.record()
        torch.cuda.synchronize()
        s = a.elapsed_time(b) / 1e3
        print(json.dumps({"primes": P, "kind": "stage-only (fwd + det + inv)", "seconds": s,
                          "dets_per_s": P * pl.node_count / s}), flush=True)
    del st
    torch.cuda.empty_cache()
    digest = None
    for P in [int(x) for x in args.full.split(",") if x]:
        c = PipelineConfig(min_primes=P)
        run_report(m, c) if digest is None else None   # warm-up once
        t0 = time.perf_counter()
        res, timings, plp = run_report(m, c)
        wall = time.perf_counter() - t0
        h = hashlib.sha256(repr(sorted(res.terms().items())).encode()).hexdigest()
        same = digest is None or h == digest
        digest = digest or h
        print(json.dumps({"primes": plp.prime_count, "kind": "full run_report", "seconds": wall,
                          "stages_s": timings.as_dict(), "dets_per_s": plp.prime_count * plp.node_count / wall,
                          "result_sha256": h, "same_result_as_first": same}), flush=True)
        if not same:
            sys.exit("result changed with the prime count")


if __name__ == "__main__":
    main()
