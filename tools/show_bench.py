import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d[k] for k in ("value","grid_dets_per_s","ms_per_step","gpu_launches")})
print("frac", d["roofline"]["frac"], d["roofline"]["frac_vs_imadwide_ceiling"], "e2e", d["e2e"]["value"], d["roofline"]["det_ms_per_step"])
for r in d.get("poly_e2e") or []: print(r["config"], round(r["seconds"],4), r.get("reference_cpu_s"), {k: round(v,4) for k,v in r["stages_s"].items()})
if "cpu_baseline" in d: print(d["cpu_baseline"]["sample"])
print(d["clocks"])
