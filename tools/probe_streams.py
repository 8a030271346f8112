"""Probe: views/s of 8-view batches on one stream vs alternating over 2-3
streams (does overlapping latency-bound sort/projection with the issue-bound
compositor pay?).  Dev tool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17338_b200 import raster, scenes
s = scenes.psi_decode_scene(352, limit=1_000_000)
cams = scenes.orbit_ring(s, count=96, size=512)
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams[:8], concurrency=8)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.3) + 65536
out = torch.empty((len(cams), 512, 512, 4), dtype=torch.float32, device="cuda")
for nstreams in (1, 2, 3, 1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        main = torch.cuda.current_stream()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(main)
        for st in streams:
            st.wait_stream(main)
        for k in range(0, len(cams), 8):
            st = streams[(k // 8) % nstreams]
            with torch.cuda.stream(st):
                raster.render_views(s, cams[k:k + 8], out=out[k:k + 8], concurrency=8)
        for st in streams:
            main.wait_stream(st)
        ev1.record(main)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    print(f"streams={nstreams} views/s={len(cams) / ms * 1e3:.0f} ms={ms:.2f}")
