import sys, time, torch
sys.path.insert(0, ".")
from paper_2010_12117_b200 import find_fourier_primes, native
for start in (10**9, 2**30 + 1):
    spec = find_fourier_primes(8, 1, start=start, min_count=1)[0]
    ctx = native.prime_context(spec)
    r, n = 40, 65536
    grids = torch.randint(0, spec.p, (r * r, n), dtype=torch.int64, device="cuda").to(torch.int32)
    ids = torch.arange(r * r, dtype=torch.int32, device="cuda")
    det = torch.empty(n, dtype=torch.int32, device="cuda")
    scratch = native.scratch_tensor(native.det_scratch_bytes(r, n))
    native.det_batch(ctx, grids, n, ids, r, 0, n, det, scratch); torch.cuda.synchronize()
    t = time.perf_counter(); native.det_batch(ctx, grids, n, ids, r, 0, n, det, scratch); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(spec.p, "%.1f M dets/s" % (n / dt / 1e6))
