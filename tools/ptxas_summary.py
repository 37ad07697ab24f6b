"""Registers / stack / spills per kernel from a ptxas -v log (csrc/build/*.ptxas.txt).

    python tools/ptxas_summary.py paper_2010_12117_b200/csrc/build/det.ptxas.txt [name-filter]
"""
import re
import subprocess
import sys


def main():
    path = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    cur = None
    rows = {}
    for line in open(path):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
            rows[cur] = {}
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            rows[cur]["regs"] = int(m.group(1))
    names = list(rows)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    for n, d in zip(names, dem):
        if filt in d:
            r = rows[n]
            print("%4s regs %4s stack %3s/%3s spill  %s" % (r.get("regs"), r.get("stack"), r.get("spill_st"),
                                                           r.get("spill_ld"), d.split("(")[0]))


if __name__ == "__main__":
    main()
