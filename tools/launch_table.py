"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9}
for r in rows[1:]:
    name = r[ik].split("(")[0][:60]
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    agg[name][r[im]] += v
    if r[im] == "gpu__time_duration.sum":
        cnt[name] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print("%-60s %6s %10s %7s %10s %10s %8s" % ("kernel", "n", "ms", "share", "MB read", "MB write", "GB/s"))
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = a["gpu__time_duration.sum"]
    rd, wr = a.get("dram__bytes_read.sum", 0), a.get("dram__bytes_write.sum", 0)
    print("%-60s %6d %10.3f %6.1f%% %10.1f %10.1f %8.0f" % (name, cnt[name], t * 1e3, 100 * t / tot, rd / 1e6, wr / 1e6,
                                                          (rd + wr) / t / 1e9 if t else 0))
