#!/bin/bash
# Quick GPU iteration: parity tests + kernel throughput for LPM 8 and 16 + bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for lpm in 8 16; do
  PDB_OCT_LPM=$lpm timeout 300 python tools/det_bench.py --r 16,40 --nodes 1048576 --fused > gpurun_out/det_bench_lpm$lpm.json 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log
