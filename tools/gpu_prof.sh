#!/bin/bash
# ncu --set full of the det kernel (fused C5 and staged r=16) + the bench launch list.
# Text dumps (details/raw csv) are written next to each report so the numbers
# survive even if a large .ncu-rep is not pulled back.
#   tools/gpu_prof.sh [kernel-regex] [tag]
K=${1:-det_gj_kernel}
T=${2:-gj}
mkdir -p gpurun_out
prof() {  # name, command...
  local name=$1; shift
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_${T}_$name -f "$@" \
    > gpurun_out/ncu_${T}_$name.log 2>&1
  ncu -i gpurun_out/prof_${T}_$name.ncu-rep --page details --csv > gpurun_out/prof_${T}_${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_${T}_$name.ncu-rep --page raw --csv > gpurun_out/prof_${T}_${name}_raw.csv 2>/dev/null
}
prof fused python tools/det_bench.py --r "" --nodes 262144 --fused --reps 1
prof r16 python tools/det_bench.py --r 16 --nodes 262144 --reps 1
if [ -z "$NO_LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_${T}.log 2>&1
fi
tail -n 2 gpurun_out/ncu_${T}_fused.log gpurun_out/ncu_${T}_r16.log
