"""Probe: single-view render() calls per second (the drop-in API) and the
device time of one-view batches, on the cfg3 scene (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig
s = scenes.psi_decode_scene(352, limit=1_000_000)
cams = scenes.orbit_ring(s, count=100, size=512)
for mode in ("exact", "fast"):
    cfg = RenderConfig(exp_mode=mode)
    for c in cams[:5]:
        raster.render(s, c, config=cfg)
    t0 = time.perf_counter()
    for c in cams[:60]:
        raster.render(s, c, config=cfg)
    dt = time.perf_counter() - t0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for c in cams[:60]:
        raster.render_views(s, [c], config=cfg)
    ev1.record()
    torch.cuda.synchronize()
    print(f"{mode}: render() {60 / dt:.0f} calls/s; one-view batches {ev0.elapsed_time(ev1) / 60:.3f} ms/view")
