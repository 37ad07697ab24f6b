import sys, time
sys.path.insert(0, ".")
from paper_2010_12117_b200 import run_report, workloads, PipelineConfig
m, _ = workloads.c3()
cfg = PipelineConfig(prime_start=2**61)
run_report(m, cfg)
t = time.perf_counter(); res, tm, pl = run_report(m, cfg); print("wide C3", pl.prime_count, "primes", time.perf_counter() - t, tm)
