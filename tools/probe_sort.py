"""Probe: render a few 16-view batches of the cfg3 workload (for ncu captures of
steady-state sort/composite launches; dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig
cfg = RenderConfig(exp_mode=os.environ.get("G6R_PROBE_EXP", "fast"))
s = scenes.psi_decode_scene(352, limit=1_000_000)
B = int(os.environ.get("G6R_PROBE_BATCH", "16"))
cams = scenes.orbit_ring(s, count=4 * B, size=512)
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams[:B], concurrency=B, config=cfg)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.5) + 65536
for k in range(3):
    raster.render_views(s, cams[B * k:B * k + B], concurrency=B, config=cfg)
torch.cuda.synchronize()
print("ok")
