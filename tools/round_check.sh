#!/bin/bash
# Full measurement pass on the GPU box: GPU tests, smoke, default bench line,
# end-to-end configs, ncu launch list of the bench command.
#   tools/round_check.sh TAG
T=${1:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
tail -2 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; cat gpurun_out/bench_$T.json; tail -2 gpurun_out/bench_$T.err
timeout 900 python tools/e2e_bench.py --configs c1,c2,c2w,c3,c4a,c4b,c5 > gpurun_out/e2e_$T.jsonl 2>&1; cut -c1-200 gpurun_out/e2e_$T.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_$T.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$T.csv 2>&1 | head -12
