"""Probe (dev tool): where the compositor's time goes on the cfg3 workload.

1. every view of the bench's 100-view orbit rendered alone (1 view per
   launch, profiler on): per-view composite ms -> spread across the orbit;
2. the bench's first 20 views and 20 views spread over the orbit, in batches
   of 10/16/20: composite ms per view (one stream, profiler on).
Run twice with G6R_SCHED=0/1 to A/B the compositor work order."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2505_17338_b200 import _native as nat
from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig

cfg = RenderConfig(exp_mode=os.environ.get("G6R_PROBE_EXP", "fast"))
s = scenes.psi_decode_scene(352, limit=1_000_000)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
lo, hi = s.mu_p.min(axis=0), s.mu_p.max(axis=0)
cams = bench.orbit_from_bbox(lo, hi, 100, 512)
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams[:16], config=cfg)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.6) + 65536


def timed(views, batch):
    prof = nat.Profiler(len(views))
    raster.render_views(s, views, config=cfg, concurrency=batch)   # warm
    raster.render_views(s, views, config=cfg, concurrency=batch, profiler=prof)
    torch.cuda.synchronize()
    ms, nv = prof.read()
    prof.close()
    return {k: v / nv for k, v in ms.items()}


out = {"sched": os.environ.get("G6R_SCHED", "1")}
per = [timed([c], 1)["composite"] for c in cams]
out["single_view_composite_ms"] = {"min": min(per), "median": float(np.median(per)),
                                   "max": max(per), "first20_mean": float(np.mean(per[:20])),
                                   "all_mean": float(np.mean(per))}
for name, views in (("first20", cams[:20]), ("spread20", cams[::5])):
    for b in (10, 16, 20):
        out[f"{name}_b{b}"] = timed(views, b)
out["all100_b16"] = timed(cams, 16)
print(json.dumps(out))
