"""Probe: host enqueue time vs device time of render_views (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_17338_b200 import raster, scenes, _native as nat
s = scenes.psi_decode_scene(352, limit=1_000_000)
cams = scenes.orbit_ring(s, count=64, size=512)
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams[:8], concurrency=8)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.5) + 65536
out = torch.empty((64, 512, 512, 4), device="cuda")
for batch in (1, 4, 8):
    for prof in (False, True):
        p = nat.Profiler(64) if prof else None
        raster.render_views(s, cams, concurrency=batch, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        raster.render_views(s, cams, concurrency=batch, out=out, profiler=p)
        t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
        st = p.read()[0] if p else {}
        print(f"batch={batch} prof={prof} enqueue_ms={1e3*(t1-t0):.2f} gpu_ms={e0.elapsed_time(e1):.2f} wall_ms={1e3*(t2-t0):.2f} views/s={64/(e0.elapsed_time(e1)/1e3):.0f} stages={ {k: round(v/64,4) for k,v in st.items()} }")
