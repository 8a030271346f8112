"""Summarise an ncu report into profiles/ncu_summary.json (dev tool).

Usage: python tools/ncu_summary.py <report.ncu-rep> <views_per_launch> [out.json]
Per kernel (first capture of each name): duration, DRAM bytes, L2 hit rate,
registers, occupancy, issued IPC, instructions.  `composite_dram_bytes_per_launch`
(per view) feeds bench.py's roofline.traffic."""
import csv, io, json, subprocess, sys

rep, views = sys.argv[1], int(sys.argv[2])
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_summary.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_MB",
        "dram__bytes_write.sum": "dram_write_MB", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
        "launch__registers_per_thread": "registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "sm__inst_executed.avg.per_cycle_active": "ipc_active",
        "smsp__inst_executed.sum": "warp_instructions",
        "launch__grid_size": "grid", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct"}
units = rows[1]
res = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("g6r::", "")
    if name in res:
        continue
    ent = {}
    for k, v in want.items():
        if k not in d:
            continue
        x = float(d[k].replace(",", "")) if d[k] not in ("", "n/a") else None
        u = units[h.index(k)]
        if x is not None and k.startswith("dram__bytes"):
            x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(u, 1.0)
        if x is not None and k == "gpu__time_duration.sum":
            x = x * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
        ent[v] = x
    res[name] = ent
summary = {"report": rep, "views_per_launch": views, "kernels": res}
comp = next((v for k, v in res.items() if k.startswith("k_composite")), None)
if comp and comp.get("dram_read_MB") is not None:
    summary["composite_dram_bytes_per_launch"] = (comp["dram_read_MB"] + comp["dram_write_MB"]) * 1e6 / views
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
