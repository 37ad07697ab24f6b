#!/bin/bash
# One iteration on the GPU box: parity tests, then kernel throughput for the
# library variants given as arguments (default: the main build), then bench.
#   tools/gpu_iter.sh [variant.so ...]      (variants live in paper_2010_12117_b200/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
R=${DET_R:-16,40}
timeout 300 python tools/det_bench.py --r $R --nodes 1048576 --fused > gpurun_out/det_bench_main.json 2>&1
echo "== main"; cat gpurun_out/det_bench_main.json | python -c "import json,sys; d=json.load(sys.stdin); [print(k, round(v['dets_per_s']/1e6,2) if isinstance(v,dict) else v) for k,v in d.items()]"
for v in "$@"; do
  # v = <library suffix or "main">, built with make BUILD=build_<v> OUT=../libpolydet_b200_<v>.so EXTRA=-D...
  # optional @W forces W warps per CTA, e.g. main@4
  warps=""
  [[ "$v" == *@* ]] && { warps=${v##*@}; v=${v%@*}; }
  lib=$v
  libpath=paper_2010_12117_b200/libpolydet_b200.so
  [ "$lib" != "main" ] && libpath=paper_2010_12117_b200/libpolydet_b200_$lib.so
  out=gpurun_out/det_bench_${lib}_${warps:-def}.json
  PDB_LIBRARY=$libpath PDB_GJ_WARPS=$warps timeout 300 python tools/det_bench.py --r $R --nodes 1048576 --fused > $out 2>&1
  echo "== $v"; python -c "import json,sys; d=json.load(open('$out')); [print(k, round(v['dets_per_s']/1e6,2) if isinstance(v,dict) else v) for k,v in d.items()]" || tail -5 $out
done
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
  cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
fi
