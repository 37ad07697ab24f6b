#!/bin/bash
# One GPU session: parity tests, kernel bench, full bench, ncu captures.
# usage: tools/gpu_check.sh [quick]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/det_bench.py --r 4,8,16,40 --nodes 1048576 --fused > gpurun_out/det_bench.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "$1" != "quick" ]; then
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:det_octet -c 1 -o gpurun_out/prof_octet_staged -f python tools/det_bench.py --r 40 --nodes 65536 --reps 1 > gpurun_out/ncu1.log 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:det_octet -c 1 -o gpurun_out/prof_octet_fused -f python tools/det_bench.py --r "" --nodes 262144 --fused --reps 1 > gpurun_out/ncu2.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/det_bench.json; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
