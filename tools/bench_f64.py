import sys, time, torch
sys.path.insert(0, '.')
from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig
s = scenes.psi_decode_scene(352, limit=1_000_000)
cams = scenes.orbit_ring(s, count=64, size=512)
cfg = RenderConfig(precision="f64")
prep = raster.prepare_scene(s)
_, c = raster.render_views(s, cams[:8], config=cfg); torch.cuda.synchronize()
prep.entry_hint = int(c[:, 1].max().item() * 1.3) + 65536
out = torch.empty((64, 512, 512, 4), dtype=torch.float64, device="cuda")
raster.render_views(s, cams, config=cfg, out=out); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); raster.render_views(s, cams, config=cfg, out=out); e1.record(); torch.cuda.synchronize()
print("f64 views/s", 64 / e0.elapsed_time(e1) * 1e3)
