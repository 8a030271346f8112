"""Probe: per-launch device intervals with G6R_TRACE=1 (dev tool)."""
import os, sys, collections
os.environ["G6R_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_17338_b200 import raster, scenes, _native as nat
from paper_2505_17338_b200.raster import RenderConfig
cfg = RenderConfig(exp_mode=os.environ.get("G6R_PROBE_EXP", "fast"))
s = scenes.psi_decode_scene(352, limit=1_000_000)
cams = scenes.orbit_ring(s, count=64, size=512)
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams[:8], concurrency=8, config=cfg)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.5) + 65536
for batch in (16, 8):
    raster.render_views(s, cams, concurrency=batch, pipeline=False, config=cfg); torch.cuda.synchronize()
    nat.load().g6r_trace_dump(b"/tmp/trace_warm.csv")
    raster.render_views(s, cams, concurrency=batch, pipeline=False, config=cfg); torch.cuda.synchronize()
    path = f"gpurun_out/trace_b{batch}.csv"
    nat.load().g6r_trace_dump(path.encode())
    agg = collections.defaultdict(list)
    for line in open(path).read().splitlines()[1:]:
        k, v = line.split(","); agg[k].append(float(v))
    tot = sum(sum(v) for v in agg.values())
    print(f"batch={batch} total_ms={tot:.2f} per_view_ms={tot/len(cams):.3f}")
    for k, v in agg.items():
        print(f"   {k:10s} n={len(v):3d} mean_ms={sum(v)/len(v):.4f} share={sum(v)/tot*100:5.1f}%")
