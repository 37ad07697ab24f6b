"""Aggregate an ncu report's per-SASS counters by CUDA source line.

    python tools/ncu_lines.py report.ncu-rep path/to/obj.o [top] [kernel-substring]

ncu's CSV source page has no source correlation, so this joins it with
`nvdisasm -g` of the object's cubin: SASS offset -> (file, line) from the
line-info comments, ncu address - kernel base -> offset.
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def ncu_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    kernel = lines[0].split('","')[1].rstrip('",') if lines[0].startswith('"Kernel Name"') else ""
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    return kernel, list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def line_map(obj, want):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=tmp, capture_output=True)
    cub = next(Path(tmp).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-gi", "-c", str(cub)], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    loc = None
    for ln in sass.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = funcs.setdefault(m.group(1), {})
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m and "inlined at" in ln:   # -gi: the last (outermost) frame names the caller's line
            continue
        if m:
            loc = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and cur is not None and loc:
            cur[int(m.group(1), 16)] = loc + (_opcode(m.group(2)),)
    cands = [f for f in funcs if all(w in f for w in want)]
    return funcs, cands


def _opcode(text):
    w = text.split()
    return (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "")).split(".")[0]


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    rep, obj = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    want = sys.argv[4].split(",") if len(sys.argv) > 4 else ["det_gj_kernel", "FusedSrc"]
    kernel, rows = ncu_rows(rep)
    funcs, cands = line_map(obj, want)
    if not cands:
        sys.exit("no function matches %s" % want)
    # choose the candidate whose instruction count matches the report
    n = len(rows)
    fn = min(cands, key=lambda f: abs(len(funcs[f]) - n))
    lmap = funcs[fn]
    base = int(rows[0]["Address"], 16)
    # the object must be the build that was profiled: compare opcodes address by address
    same = sum(1 for r in rows if lmap.get(int(r["Address"], 16) - base, ("", 0, ""))[2] == _opcode(r["Source"]))
    if same < 0.95 * len(rows):
        sys.exit("object does not match the profiled build (%d of %d opcodes agree)" % (same, len(rows)))
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    tot = [0.0, 0.0, 0.0]
    reasons = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    why = collections.defaultdict(collections.Counter)
    for r in rows:
        off = int(r["Address"], 16) - base
        loc = lmap.get(off, ("?", 0, ""))[:2]
        v = (num(r["Thread Instructions Executed"]), num(r["Warp Stall Sampling (All Samples)"]),
             num(r["Instructions Executed"]))
        for i in range(3):
            agg[loc][i] += v[i]
            tot[i] += v[i]
        for c in reasons:
            why[loc][c[6:]] += num(r[c])
    print("kernel:", kernel)
    print("function:", fn, " sass rows:", n, " mapped:", len(lmap))
    print("%-28s %10s %8s %8s" % ("file:line", "thr-inst%", "stall%", "warp-inst%"))
    for loc, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        top3 = ", ".join("%s %.0f%%" % (k, 100 * n / max(v[1], 1)) for k, n in why[loc].most_common(3))
        print("%-28s %9.2f%% %7.2f%% %8.2f%%   %s" % ("%s:%d" % loc, 100 * v[0] / tot[0], 100 * v[1] / max(tot[1], 1),
                                                     100 * v[2] / tot[2], top3))


if __name__ == "__main__":
    main()
