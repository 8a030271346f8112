"""Per-kernel table of the bench's own views (dev tool) -> profiles/<tag>_kernels.json.

Input: the ncu launch list of tools/probe_bench_views.py (gpu__time_duration,
dram bytes read/write per launch, --clock-control none) and optionally the
`--set full` summary written by tools/ncu_summary.py.  The profiled pass is
the last `batches` batches of g6r kernels in the list (the probe renders the
views once more, one stream, at the end).  Output per kernel: launches per
batch, mean duration per launch, DRAM bytes per launch, the kernel's share of
the pass; plus the whole path's DRAM bytes per view, which bench.py turns into
the DRAM-counter roofline fraction beside the algorithmic one.

    python tools/launch_table.py launches.csv views batches out.json [full_summary.json]
"""
import collections
import csv
import json
import sys

path, views, batches, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
full = json.load(open(sys.argv[5])) if len(sys.argv) > 5 else None
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value",
                                            "Metric Unit"))
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").replace("g6r::", "")})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
launches = [d for d in per.values() if not d["name"].startswith("at::")]
# the profiled pass: from the last `batches` k_clear launches on
clears = [i for i, d in enumerate(launches) if d["name"] == "k_clear"]
tail = launches[clears[-batches]:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in tail:
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot_us = sum(a[1] for a in agg.values())
tot_bytes = sum(a[2] for a in agg.values())
table = {k: {"launches_per_batch": a[0] / batches, "mean_us": a[1] / a[0],
             "dram_MB_per_launch": a[2] / a[0] / 1e6, "share": a[1] / tot_us,
             "us_per_view": a[1] / views}
         for k, a in sorted(agg.items(), key=lambda x: -x[1][1])}
res = {"source": path, "views": views, "batches": batches, "views_per_launch": views / batches,
       "kernels": table, "pass_us_per_view": tot_us / views,
       "dram_bytes_per_view": tot_bytes / views}
comp = [k for k in table if k.startswith("k_composite")]
if comp:
    c = agg[comp[0]]
    res["composite_dram_bytes_per_launch"] = c[2] / c[0]
if full:
    res["full"] = full.get("kernels", full)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: round(v["us_per_view"], 2) for k, v in table.items()}))
print("pass us/view", round(tot_us / views, 1), "dram MB/view", round(tot_bytes / views / 1e6, 1))
