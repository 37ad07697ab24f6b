"""Issue-cost breakdown of det_gj_kernel by phase (fill / P / M / T / other).

    python tools/ncu_phases.py report.ncu-rep obj.o FILL,P_FIRST,P_LAST,M,T [nodes]

(FILL, M and T may be several lines joined by '+'.)

The line numbers are det_gj.cuh lines of the kernel body (fill call, first and
last line of the pivot-block phase, M-pass call, T-pass call); an instruction
belongs to a phase when any frame of its inlining chain (nvdisasm -gi) is on
one of those lines, so code inlined through the block lambda is attributed
too.  Weights model the measured B200 issue cost per warp instruction
(tools/microbench/pipes.cu): IMAD.WIDE ~4.2 cycles, IMAD.HI ~4, other IMAD
forms 2, everything else 1; the sum over all SASS reproduces the fused
kernel's elapsed SMSP cycles to a few per cent.
"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_lines import _opcode, ncu_rows, num  # noqa: E402

W = {"IMAD.WIDE.U32": 4.2, "IMAD.WIDE": 4.2, "IMAD.HI.U32": 4.0}


def chains(obj, want):
    """function -> {offset: (opcode, [det_gj.cuh lines of the inlining chain])}"""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=tmp, capture_output=True)
    cub = next(Path(tmp).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-gi", "-c", str(cub)], capture_output=True, text=True).stdout
    funcs, cur, pend, loc = {}, None, [], []
    for ln in sass.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = funcs.setdefault(m.group(1), {})
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            if Path(m.group(1)).name == "det_gj.cuh":
                pend.append(int(m.group(2)))
            if m.group(3) and Path(m.group(3)).name == "det_gj.cuh":
                pend.append(int(m.group(4)))
            if not m.group(3):
                loc, pend = pend, []
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and cur is not None:
            cur[int(m.group(1), 16)] = (_opcode(m.group(2)), loc)
    cands = [f for f in funcs if all(w in f for w in want)]
    return funcs, cands


def main():
    rep, obj = sys.argv[1], sys.argv[2]
    # each field may list several call lines joined by '+' (e.g. the M pass has one call per variant)
    FILL, P0, P1, MP, TP = ({int(y) for y in x.split("+")} for x in sys.argv[3].split(","))
    P0, P1 = min(P0), max(P1)
    nd = int(sys.argv[4]) if len(sys.argv) > 4 else 262144
    _, rows = ncu_rows(rep)
    funcs, cands = chains(obj, ["det_gj_kernel", "FusedSrc"])
    base = int(rows[0]["Address"], 16)

    def agree(f):
        return sum(1 for r in rows if funcs[f].get(int(r["Address"], 16) - base, ("",))[0] == _opcode(r["Source"]))
    fn = max(cands, key=agree)
    if agree(fn) < 0.95 * len(rows):
        sys.exit("object does not match the profiled build")
    lmap = funcs[fn]

    def phase(lines):
        if TP & set(lines):
            return "T"
        if MP & set(lines):
            return "M"
        if FILL & set(lines):
            return "fill"
        if any(P0 <= x <= P1 for x in lines):
            return "P"
        return "other"
    ph = collections.defaultdict(collections.Counter)
    stall = collections.defaultdict(collections.Counter)
    reasons = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    for r in rows:
        _, lines = lmap.get(int(r["Address"], 16) - base, ("", []))
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r["Source"])
        op = m.group(2) if m else "?"
        w = W.get(op, 2.0 if op.startswith("IMAD") else 1.0)
        ph[phase(lines)][op] += w * num(r["Instructions Executed"])
        stall[phase(lines)]["ALL"] += num(r.get("Warp Stall Sampling (All Samples)", "0"))
        for c in reasons:
            stall[phase(lines)][c[6:]] += num(r[c])
    tot = sum(sum(c.values()) for c in ph.values())
    for k, c in sorted(ph.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(c.values())
        print("%-6s %5.1f%%  %7.0f weighted warp-inst/det   top: %s" % (
            k, 100 * s / tot, s / nd, ", ".join("%s %.0f" % (o, v / nd) for o, v in c.most_common(6))))
    print("total weighted SMSP-cycles per det (sum over SMSPs):", tot / nd)
    sall = sum(c["ALL"] for c in stall.values()) or 1
    print("warp-state samples per phase (share of all samples; top reasons within the phase):")
    for k, c in sorted(stall.items(), key=lambda kv: -kv[1]["ALL"]):
        top = [(n, v) for n, v in c.most_common() if n != "ALL"][:5]
        print("%-6s %5.1f%%   %s" % (k, 100 * c["ALL"] / sall,
                                     ", ".join("%s %.0f%%" % (n, 100 * v / max(c["ALL"], 1)) for n, v in top)))


if __name__ == "__main__":
    main()
