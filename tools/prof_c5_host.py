import cProfile, pstats, sys, time
sys.path.insert(0, ".")
from paper_2010_12117_b200 import run_report, workloads
m, cfg = workloads.c5()
run_report(m, cfg)
pr = cProfile.Profile(); pr.enable()
t = time.perf_counter(); run_report(m, cfg); print("wall", time.perf_counter() - t)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
