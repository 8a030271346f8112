"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum,... --csv) per
kernel: launches, total and mean duration, share of the total, DRAM bytes per
launch (dev tool).   python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9}
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values()) or 1.0
print(f"{'kernel':44s} {'n':>4s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s} {'MB/launch':>9s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} {a[0]:4d} {a[1]:10.1f} {a[1] / a[0]:9.1f} {a[1] / tot:6.3f} {a[2] / a[0] / 1e6:9.2f}")
