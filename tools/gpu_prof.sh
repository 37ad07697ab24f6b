#!/bin/bash
# ncu --set full of the det kernel (fused C5 and staged r) + the bench launch list.
#   tools/gpu_prof.sh [kernel-regex] [tag]
K=${1:-det_gj_kernel}
T=${2:-gj}
mkdir -p gpurun_out
timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_${T}_fused -f \
  python tools/det_bench.py --r "" --nodes 262144 --fused --reps 1 > gpurun_out/ncu_${T}_fused.log 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_${T}_r16 -f \
  python tools/det_bench.py --r 16 --nodes 262144 --reps 1 > gpurun_out/ncu_${T}_r16.log 2>&1
if [ -z "$NO_LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_${T}.log 2>&1
fi
tail -n 2 gpurun_out/ncu_${T}_fused.log gpurun_out/ncu_${T}_r16.log
