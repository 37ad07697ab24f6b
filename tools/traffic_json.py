"""Summarise one `ncu --set full` capture of the fused det kernel into the JSON
bench.py reads for the roofline `traffic` field and the `ncu` summary.

    python tools/traffic_json.py profiles/ncu/prof_<tag>_fused_raw.csv \
        profiles/ncu/prof_<tag>_fused.ncu-rep > profiles/ncu/det_traffic_r01.json

The weighted issue model (tools/ncu_phases.py, tools/microbench/pipes.cu)
charges IMAD.WIDE ~4.2 and IMAD.HI ~4 issue cycles, other IMAD forms 2, the
rest 1; `issue_model_cycles_frac` is its total over the SMSPs' elapsed cycles.
"""
import collections
import csv
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_lines import ncu_rows, num  # noqa: E402

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}
W = {"IMAD.WIDE.U32": 4.2, "IMAD.WIDE": 4.2, "IMAD.HI.U32": 4.0}


def main():
    raw, rep = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(raw)))
    d = {h: (v, u) for h, u, v in zip(*rows[:3])}

    def val(k):
        v, u = d[k]
        return float(v.replace(",", "")) * UNITS.get(u, 1)

    # optional: nodes in the profiled launch and nodes per coefficient slab (the
    # pruned C5 launch covers whole kept last-axis rows of 176 nodes)
    nodes = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
    row = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    slab = 5 * 1600 * 4
    algo = nodes // row * slab + 8 * nodes
    _, srows = ncu_rows(rep)
    mix = collections.Counter()
    for r in srows:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r["Source"])
        mix[m.group(2) if m else "?"] += num(r["Instructions Executed"])
    weighted = sum(n * W.get(op, 2.0 if op.startswith("IMAD") else 1.0) for op, n in mix.items())
    smsps = 148 * 4
    out = {
        "kernel": "det_gj_kernel<FusedSrc,1,16,P31=0,RPC=40> (C5 prime 0, 40x40, fused DFT-8 fill)",
        "source": "%s (ncu --set full --clock-control none, tools/gpu_prof.sh)" % raw,
        "command": "python tools/det_bench.py --r '' --nodes 262144 %s --reps 1" % ("--pruned" if row != 256 else "--fused"),
        "nodes_per_launch": nodes,
        "dram_read_bytes": val("dram__bytes_read.sum"),
        "dram_write_bytes": val("dram__bytes_write.sum"),
        "algorithmic_bytes": algo,
        "algorithmic_note": "one [E=5][k=1600] u32 coefficient slab per outer index o (%d nodes of the launch), "
                            "+ num/den u32 per node" % row,
        "dram_bytes_per_node": (val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / nodes,
        "duration_s": val("gpu__time_duration.sum"),
        "pipes_pct_of_peak": {
            "fma": val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fmaheavy": val("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "alu": val("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "lsu": val("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "tensor": 0.0, "fp64": 0.0,
        },
        "issue_active_pct": val("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        "warp_instructions": sum(mix.values()),
        "warp_instructions_per_det": sum(mix.values()) / nodes,
        "issue_model_cycles_per_det": weighted / nodes,
        "issue_model_cycles_frac": weighted / smsps / val("sm__cycles_elapsed.avg"),
        "top_ops_per_det": {op: n / nodes for op, n in mix.most_common(8)},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
