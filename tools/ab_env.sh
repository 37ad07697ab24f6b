#!/bin/bash
# A/B of one environment switch on the det kernel, alternating runs in one box call:
#   tools/ab_env.sh "PDB_GJ_NO_PAIR=1" [rounds]
# prints M dets/s of det_bench (staged r=40, fused C5 incl. the pruned launch) per run.
mkdir -p gpurun_out
V=$1
N=${2:-3}
R=${DET_R:-40}
for i in $(seq 1 $N); do
  for arm in base var; do
    if [ $arm = base ]; then
      timeout 300 python tools/det_bench.py --r $R --nodes 1048576 --pruned > gpurun_out/ab_${arm}_$i.json 2>&1
    else
      env $V timeout 300 python tools/det_bench.py --r $R --nodes 1048576 --pruned > gpurun_out/ab_${arm}_$i.json 2>&1
    fi
    python - "$arm" "gpurun_out/ab_${arm}_$i.json" <<'EOF'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], " ".join("%s=%.2f" % (k, v["dets_per_s"] / 1e6) for k, v in d.items() if isinstance(v, dict) and "dets_per_s" in v))
except Exception as e:
    print(sys.argv[1], "failed", e, open(sys.argv[2]).read()[-400:])
EOF
  done
done
