"""Executed-instruction mix (by opcode) of the SASS that maps to given source lines.

    python tools/ncu_opmix.py report.ncu-rep obj.o kernel-substrings line[,line...]
"""
import collections
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_lines import line_map, ncu_rows, num  # noqa: E402


def main():
    rep, obj, want, lines = sys.argv[1], sys.argv[2], sys.argv[3].split(","), set(int(x) for x in sys.argv[4].split(","))
    _, rows = ncu_rows(rep)
    funcs, cands = line_map(obj, want)
    fn = min(cands, key=lambda f: abs(len(funcs[f]) - len(rows)))
    lmap = funcs[fn]
    base = int(rows[0]["Address"], 16)
    mix = collections.Counter()
    tot = 0.0
    for r in rows:
        loc = lmap.get(int(r["Address"], 16) - base, ("?", 0))
        if loc[1] not in lines:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r["Source"])
        op = m.group(2) if m else "?"
        n = num(r["Instructions Executed"])
        mix[op] += n
        tot += n
    print("warp instructions executed on lines %s: %.4g" % (sorted(lines), tot))
    for op, n in mix.most_common(25):
        print("  %-24s %6.2f%%  %.4g" % (op, 100 * n / tot, n))


if __name__ == "__main__":
    main()
