"""Small end-to-end workload for compute-sanitizer (dev tool).

Exercises every kernel family through the public API at cfg1 size (10k
Gaussians, 128x128): render (entry-sort path: ordered projection, onesweep,
ranges; f32 exact, f64), render_views (splat sort + tile partition + the
longest-first compositor schedule, fast and exact, runs exported), RGBA8
frames, the kernel-module adapter (stage1/2, composite, deterministic
composite_backward), render_backward, the loss + Adam of the fine-tune loop,
G6DS decode and the group filter.  Checks nothing itself: the sanitizer log
is the result (tools/sanitize.sh).

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_17338_b200 import diffrender, kernels, raster, scenes, sceneio  # noqa: E402
from paper_2505_17338_b200.raster import RenderConfig  # noqa: E402
from paper_2505_17338_b200.scene import filter_scene  # noqa: E402

n = int(os.environ.get("G6R_SAN_N", "10000"))
size = int(os.environ.get("G6R_SAN_SIZE", "128"))
s = scenes.random_scene(np.random.default_rng(0), n)
cams = scenes.orbit_ring(s, count=6, size=size)
cam = scenes.benchmark_camera(s, size, size)

st = raster.render_with_state(s, cam)                                   # ordered path, f32
st64 = raster.render_with_state(s, cam, config=RenderConfig(precision="f64"))
raster.render(s, cam, group_mask=(2, 5))
prep = raster.prepare_scene(s)
T = ((size + 15) // 16) ** 2
es = torch.empty((len(cams), prep.entry_hint), dtype=torch.int32, device="cuda")
ts = torch.empty((len(cams), T + 1), dtype=torch.int64, device="cuda")
raster.render_views(s, cams, entry_splat=es, tile_starts=ts)             # splat sort + partition
raster.render_views(s, cams, config=RenderConfig(exp_mode="fast"))
raster.render_views(s, cams, config=RenderConfig(tile_size=8))           # non-16 tiles
raster.render_frames_u8(s, cams[:3], background=(0.1, 0.2, 0.3))
raster.render_views(s, cams[:2], capacity=64)                            # overflow path

sp = st64.splats
en = st64.entries
g = np.random.default_rng(1).normal(size=st64.image.shape)
rows = np.zeros((len(en.entry_splat), 9))
kernels.composite_backward(sp.means2d, sp.conics, sp.colors, sp.alphas, en.entry_splat,
                           en.tile_starts, en.tiles_x, 16, st64.final_t, st64.last_contrib, g, rows)
img = np.zeros((size, size, 4), np.float32)
ft = np.ones((size, size), np.float32)
last = np.zeros((size, size), np.int32)
kernels.composite_forward(sp.means2d.astype(np.float32), sp.conics.astype(np.float32),
                          sp.colors.astype(np.float32), sp.alphas.astype(np.float32),
                          en.entry_splat, en.tile_starts, en.tiles_x, 16, img, ft, last)
raster.bin_splats(st.splats, cam, 16)

diffrender.render_backward(s, cam, g)
views = [(c, scenes.synthetic_target(size, size, seed=k)) for k, c in enumerate(cams[:2])]
diffrender.finetune(s, views, iters=3)

with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "s.g6ds")
    sceneio.save_scene(s, p)
    sceneio.load_scene_device(p)
raster.render(filter_scene(s, (3, 7)), cam)
torch.cuda.synchronize()
print("sanitize probe done")
