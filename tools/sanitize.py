"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck):  compute-sanitizer --tool racecheck python tools/sanitize.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2010_12117_b200 import (PipelineConfig, PrimeSpec, det_grid, executor, find_fourier_primes,  # noqa: E402
                                   run, workloads)

spec = find_fourier_primes(8, 1, start=10**9, min_count=1)[0]
rng = np.random.default_rng(0)
for r in (4, 10, 16, 40):
    grids = [rng.integers(0, spec.p, 40) for _ in range(r * r)]
    grids[0][::3] = 0                         # zero pivots -> robust path
    det_grid(grids, r, spec)
det_grid([rng.integers(0, 97, 40) for _ in range(100)], 10, PrimeSpec(97, 96, 0, 1))
m, cfg = workloads.harmonic(3, (5, 7), True)
executor.FORCE_MODE = "fused"
run(m, cfg)
executor.FORCE_MODE = "staged"
run(m, cfg)
import random  # noqa: E402
from paper_2010_12117_b200 import poly_matrix  # noqa: E402
rr = random.Random(1)
for r in (16, 40):   # compile-time-order kernels with the dense DFT-8 fill (distinct entries)
    rows = [[{(0,): rr.randint(-10**6, 10**6), (1,): rr.randint(-10**6, 10**6)} for _ in range(r)] for _ in range(r)]
    executor.FORCE_MODE = "fused"
    run(poly_matrix(rows, ("x",)))
# every axis pruned: kept-node forward passes + direct interpolation (grid_interp)
import itertools  # noqa: E402
mons = list(itertools.product(range(5), range(5)))
rows = [[{e: rr.randint(-50, 50) for e in mons if rr.random() < 0.8} for _ in range(10)] for _ in range(10)]
executor.FORCE_MODE = "fused"
run(poly_matrix(rows, ("x", "y")))
# register-radix NTTs on assorted tile shapes (TI = 1, 2..16, 32), forward and inverse
from paper_2010_12117_b200 import TwiddleTable, encode, ntt_forward_multi, ntt_inverse_multi, reduce_mod  # noqa: E402
tab = TwiddleTable(spec)
for shape in [(64,), (16, 16, 8), (256, 4), (32, 2), (128, 64)]:
    terms = {tuple(rr.randrange(n) for n in shape): rr.randint(1, 10**6) for _ in range(50)}
    t = reduce_mod(encode(terms, shape, tuple("abc"[:len(shape)])), spec)
    assert ntt_inverse_multi(ntt_forward_multi(t, tab), tab).residues.tolist() == t.residues.tolist()
executor.FORCE_MODE = None
run(*workloads.c1())
m = workloads.c1()[0]
run(m, PipelineConfig(prime_start=2**61))    # wide path
print("sanitize workload done")
