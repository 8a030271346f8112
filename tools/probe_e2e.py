"""Probe (dev tool): end-to-end render_batch (host images) on the bench's
views, against the device-resident render_views, several repetitions.

    python tools/probe_e2e.py [--views 20] [--batch 16] [--reps 5]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_17338_b200 import raster  # noqa: E402
from paper_2505_17338_b200.raster import RenderConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=20)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cfg = RenderConfig(exp_mode="fast")
s = bench.make_scene(bench.N_GAUSS)
lo, hi = s.mu_p.min(axis=0), s.mu_p.max(axis=0)
cams = bench.orbit_from_bbox(lo, hi, max(100, a.views), 512)[:a.views]
raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams, config=cfg)
torch.cuda.synchronize()
res = {"zero_copy": raster.ZERO_COPY}
for name in ("device", "e2e"):
    ts = []
    for _ in range(a.reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name == "device":
            raster.render_views(s, cams, config=cfg, concurrency=a.batch)
            torch.cuda.synchronize()
        else:
            raster.render_batch(s, cams, config=cfg, batch=a.batch)
        ts.append(time.perf_counter() - t0)
    ts = sorted(ts[1:])
    res[name] = {"views_per_s_median": a.views / ts[len(ts) // 2], "best": a.views / ts[0]}
print(json.dumps(res))
