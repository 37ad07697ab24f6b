"""Breakdown of the C5 CRT stage (device lift + host materialisation).

    python tools/prof_crt_stage.py
Runs the C5 residues of 23 primes through crt.device_lift pieces with timers.
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_12117_b200 import crt, native  # noqa: E402


def main():
    n = 256 ** 3
    P = 23
    primes = [p for p in range(10**9 + 1, 10**9 + 10**6, 2) if all(p % q for q in range(3, 32000, 2))][:P]
    dev = torch.device("cuda")
    box = torch.zeros((256, 256, 256), dtype=torch.bool)
    box[:161, :161, :161] = True
    idx = box.flatten().nonzero().squeeze(1).to(dev)
    res = torch.zeros((P, n), dtype=torch.int32, device=dev)
    for i, p in enumerate(primes):
        res[i, idx] = torch.randint(0, p, (idx.numel(),), device=dev, dtype=torch.int64).to(torch.int32)
    torch.cuda.synchronize()
    for rep in range(3):
        t0 = time.perf_counter()
        out = crt.device_lift(res, primes, n, n)
        t1 = time.perf_counter()
        tup = tuple(out)
        t2 = time.perf_counter()
        print("device_lift %.3f s, tuple() %.3f s, nonzero %d" % (t1 - t0, t2 - t1, idx.numel()))
        del out, tup
    # pieces
    host = native.host_module()
    L = native.crt_limbs(P, False)
    ix = torch.empty(n, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    native.crt_nonzero(res, P, n, n, ix, cnt)
    count = int(cnt.item()); t1 = time.perf_counter()
    limbs = torch.empty((count, L), dtype=torch.int32, device=dev)
    neg = torch.empty(count, dtype=torch.uint8, device=dev)
    wbuf = torch.zeros(1, dtype=torch.int32, device=dev)
    native.crt_mrc_sel(res, P, n, primes, ix, count, limbs, L, neg, wbuf)
    width = int(wbuf.item()); t2 = time.perf_counter()
    idx_h = np.ascontiguousarray(ix[:count].cpu().numpy())
    neg_h = np.ascontiguousarray(neg[:count].cpu().numpy()); t3 = time.perf_counter()
    lh = crt._to_host(limbs[:count, :width]); t4 = time.perf_counter()
    out = host.ints_from_limbs(lh, idx_h, neg_h, n, width); t5 = time.perf_counter()
    print("nonzero %.4f  lift %.4f  idx/neg D2H %.4f  limbs D2H %.4f (%.0f MB)  ints %.4f  (width %d)"
          % (t1 - t0, t2 - t1, t3 - t2, t4 - t3, lh.nbytes / 1e6, t5 - t4, width))


if __name__ == "__main__":
    main()
