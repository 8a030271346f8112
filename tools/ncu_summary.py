"""Summarise ncu --set full reports into profiles/ncu_summary.json (dev tool).

Usage: python tools/ncu_summary.py <views_per_launch> <out.json> <report.ncu-rep>...
Per kernel (first capture of each name): duration, DRAM bytes, L2 hit rate,
registers, occupancy, issue-slot utilisation, pipe utilisation, top stall
reasons, instructions.  `composite_dram_bytes_per_launch` (per view) feeds
bench.py's roofline.traffic."""
import csv, io, json, subprocess, sys

views, out, reps = int(sys.argv[1]), sys.argv[2], sys.argv[3:]
try:
    PEAK_GBPS = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except Exception:
    PEAK_GBPS = 6548.5
want = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_MB",
        "dram__bytes_write.sum": "dram_write_MB", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid",
        "launch__block_size": "block",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "smsp__inst_executed.sum": "warp_instructions",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct"}
scale_b = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3,
           "MB": 1.0, "GB": 1e3}
scale_t = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
res = {}
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("g6r::", "")
        if name in res:
            continue
        ent = {"report": rep}
        for k, v in want.items():
            if k not in d or d[k] in ("", "n/a"):
                continue
            x = float(d[k].replace(",", ""))
            u = units[h.index(k)]
            if k.startswith("dram__bytes"):
                x *= scale_b.get(u, 1.0)
            if k == "gpu__time_duration.sum":
                x *= scale_t.get(u, 1.0)
            ent[v] = x
        stalls = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                   float(d[k] or 0)) for k in h
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        ent["top_stalls"] = dict(sorted(stalls, key=lambda t: -t[1])[:4])
        if ent.get("duration_us") and ent.get("dram_read_MB") is not None:
            # achieved DRAM bandwidth of this capture against the measured copy peak
            gbs = (ent["dram_read_MB"] + ent["dram_write_MB"]) * 1e6 / (ent["duration_us"] * 1e-6) / 1e9
            ent["dram_GBps"] = gbs
            ent["dram_frac_of_peak"] = gbs / PEAK_GBPS
        res[name] = ent
summary = {"views_per_launch": views, "kernels": res}
comp = next((v for k, v in res.items() if k.startswith("k_composite")), None)
if comp and comp.get("dram_read_MB") is not None:
    summary["composite_dram_bytes_per_launch"] = (comp["dram_read_MB"] + comp["dram_write_MB"]) * 1e6 / views
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
