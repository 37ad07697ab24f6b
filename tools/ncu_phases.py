"""Issue-cost breakdown of det_gj_kernel by phase (fill / P / M / T / other).

    python tools/ncu_phases.py report.ncu-rep obj.o FILL,P_FIRST,P_LAST,M,T [nodes]

The line numbers are det_gj.cuh lines of the kernel body (fill call, first and
last line of the pivot-block phase, M-pass call, T-pass call).  Weights model
the measured B200 issue cost per warp instruction (tools/microbench/pipes.cu):
IMAD.WIDE ~4.2 cycles, IMAD.HI ~4, other IMAD forms 2, everything else 1; the
sum over all SASS reproduces the fused kernel's elapsed SMSP cycles.
"""
import sys, re, collections
sys.path.insert(0, __file__.rsplit('/', 1)[0])
from ncu_lines import ncu_rows, num, line_map
_, rows = ncu_rows(sys.argv[1])
funcs, cands = line_map(sys.argv[2], ["det_gj_kernel","FusedSrc"])
fn = min(cands, key=lambda f: abs(len(funcs[f]) - len(rows)))
lmap=funcs[fn]; base=int(rows[0]["Address"],16)
W={'IMAD.WIDE.U32':4.2,'IMAD.WIDE':4.2,'IMAD.HI.U32':4.0}
ph=collections.defaultdict(lambda: collections.Counter())
FILL, P0, P1, MP, TP = (int(x) for x in sys.argv[3].split(","))
def phase(line):
    if line==TP: return 'T'
    if line==MP: return 'M'
    if line==FILL: return 'fill'
    if P0<=line<=P1: return 'P'
    return 'other'
for r in rows:
    loc=lmap.get(int(r["Address"],16)-base,("?",0,""))
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r["Source"])
    op=m.group(2) if m else "?"
    w = W.get(op, 2.0 if op.startswith('IMAD') else 1.0)
    ph[phase(loc[1])][op]+= w*num(r["Instructions Executed"])
tot=sum(sum(c.values()) for c in ph.values())
nd=int(sys.argv[4]) if len(sys.argv)>4 else 262144
for k,c in sorted(ph.items(), key=lambda kv:-sum(kv[1].values())):
    s=sum(c.values())
    print("%-6s %5.1f%%  %7.0f weighted warp-inst/det   top: %s"%(k,100*s/tot,s/nd, ", ".join("%s %.0f"%(o,v/nd) for o,v in c.most_common(6))))
print("total weighted SMSP-cycles per det (sum over SMSPs):", tot/nd)
