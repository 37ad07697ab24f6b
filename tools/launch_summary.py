"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/launch_summary.py launches.csv
"""
import csv
import io
import sys


def main():
    rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
    agg = {}
    for x in csv.DictReader(io.StringIO("".join(rows))):
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = x["Kernel Name"].split("(")[0][:70]
        v = float(x["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(x["Metric Unit"], 1.0)
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print("%-72s %5s %12s %7s" % ("kernel", "n", "total us", "share"))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-72s %5d %12.1f %6.1f%%" % (k, v[0], v[1], 100 * v[1] / tot))


if __name__ == "__main__":
    main()
