"""Probe: per-batch fixed cost (launch gaps) with a tiny scene (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_17338_b200 import raster, scenes, _native as nat
for n in (1000, 100_000):
    s = scenes.random_scene(np.random.default_rng(0), n)
    cams = scenes.orbit_ring(s, count=64, size=512)
    for batch in (1, 8):
        raster.render_views(s, cams, concurrency=batch)
        torch.cuda.synchronize()
        p = nat.Profiler(64)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        raster.render_views(s, cams, concurrency=batch, profiler=p)
        e1.record(); torch.cuda.synchronize()
        st = p.read()[0]
        nb = 64 // batch
        print(f"n={n} batch={batch} per-batch ms={e0.elapsed_time(e1)/nb:.3f} stages/batch={ {k: round(v/nb,4) for k,v in st.items()} }")
