"""Summarise an ncu report's SASS source page: executed-instruction mix and
stall hot spots.

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rs = rows(rep)
    total = sum(num(r["Instructions Executed"]) for r in rs)
    samples = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rs)
    mix = collections.Counter()
    for r in rs:
        op = r["Source"].split()[0] if r["Source"] else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        mix[op] += num(r["Instructions Executed"])
    print("executed warp instructions: %.4g   stall samples: %d" % (total, samples))
    for op, n in mix.most_common(20):
        print("  %-22s %6.2f%%" % (op, 100 * n / total))
    print("\nhottest instructions (stall samples):")
    for r in sorted(rs, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]:
        print("  %s %-48s exec=%-10.3g samples=%d" % (r["Address"], r["Source"][:48],
                                                    num(r["Instructions Executed"]),
                                                    num(r["Warp Stall Sampling (All Samples)"])))


if __name__ == "__main__":
    main()
