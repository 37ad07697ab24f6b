"""Break down the CRT / result-materialisation stage of C5 on the GPU:
nonzero compaction, the lift kernel, the D2H of the used limbs and the
Python-int construction (crt.device_lift), each timed separately.

    python tools/prof_crt.py [--config c5|c3]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_12117_b200 import crt, executor, native, plan, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    a = ap.parse_args()
    m, cfg = workloads.c5() if a.config == "c5" else workloads.c3()
    pl = plan(m, cfg)
    st = executor.PrimeStages(m, pl, staged=(a.config != "c5"))
    P, n = pl.prime_count, pl.node_count
    res = torch.empty((P, n), dtype=torch.int32, device="cuda")
    for pi in range(P):
        st.step(pi)
        res[pi].copy_(st.det)
    del st
    torch.cuda.synchronize()
    primes = [s.p for s in pl.primes]
    out = {"config": a.config, "primes": P, "nodes": n}
    for rep in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        idx = torch.empty(n, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t0 = time.perf_counter()
        ev[0].record()
        native.crt_nonzero(res, P, n, n, idx, cnt)
        ev[1].record()
        count = int(cnt.item())
        L = native.crt_limbs(P)
        limbs = torch.empty((count, L), dtype=torch.int32, device="cuda")
        neg = torch.empty(count, dtype=torch.uint8, device="cuda")
        wb = torch.zeros(1, dtype=torch.int32, device="cuda")
        e2 = torch.cuda.Event(enable_timing=True)
        e2.record()
        native.crt_mrc_sel(res, P, n, primes, idx, count, limbs, L, neg, wb)
        ev[2].record()
        width = int(wb.item())
        t1 = time.perf_counter()
        h = crt._to_host(limbs[:, :width])
        ih = idx[:count].cpu().numpy()
        nh = neg.cpu().numpy()
        t2 = time.perf_counter()
        ints = native.host_module().ints_from_limbs(h, ih, nh, n, width)
        t3 = time.perf_counter()
        t4 = time.perf_counter()
        full = crt.device_lift(res, primes, n, n)
        t5 = time.perf_counter()
        assert full == ints
        out["rep%d" % rep] = {"nonzero_ms": ev[0].elapsed_time(ev[1]), "lift_kernel_ms": e2.elapsed_time(ev[2]),
                              "count": count, "width": width, "device_s": t1 - t0, "d2h_s": t2 - t1,
                              "ints_s": t3 - t2, "device_lift_s": t5 - t4,
                              "d2h_bytes": count * width * 4 + count * 9}
        del ints, full
    print(json.dumps(out))


if __name__ == "__main__":
    main()
