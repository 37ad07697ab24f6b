#!/bin/bash
# Run the default bench N times (without the polynomial and CPU legs) and keep
# one summary line per run: run-to-run spread of value / e2e / roofline frac.
N=${1:-3}
mkdir -p gpurun_out
for i in $(seq 1 $N); do
  python bench.py --no-poly --no-cpu-baseline 2>/dev/null > gpurun_out/bench_rep_$i.json
  python - "$i" <<'PY'
import json, sys
d = json.load(open("gpurun_out/bench_rep_%s.json" % sys.argv[1]))
print(json.dumps({"run": int(sys.argv[1]), "value": d["value"], "e2e": d["e2e"]["value"],
                  "frac": d["roofline"]["frac"], "peak": d["roofline"]["peak"], "clocks": d["clocks"]}))
PY
done
