"""Compositor CTA timeline (dev tool; needs the -DG6R_CTA_TRACE build):

    make -C paper_2505_17338_b200/csrc OUT_DIR=../_lib_trace EXTRA=-DG6R_CTA_TRACE
    G6R_LIBRARY=$PWD/paper_2505_17338_b200/_lib_trace/libg6r.so python tools/cta_trace.py

Renders the bench's 20 views (two 10-view batches, one stream) and prints, per
compositor launch: its span, when the last CTA started, the longest CTAs (run
length, duration), and how busy the SMs were over time (CTAs resident per SM
in 10 time slices) -- i.e. whether the launch is bound by throughput or by
its longest CTAs."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_17338_b200 import _native as nat  # noqa: E402
from paper_2505_17338_b200 import raster  # noqa: E402
from paper_2505_17338_b200.raster import RenderConfig  # noqa: E402

views = int(os.environ.get("VIEWS", "20"))
batch = int(os.environ.get("BATCH", "10"))
cfg = RenderConfig(exp_mode=os.environ.get("EXP", "fast"))
s = bench.make_scene(bench.N_GAUSS)
lo, hi = s.mu_p.min(axis=0), s.mu_p.max(axis=0)
cams = bench.orbit_from_bbox(lo, hi, 100, 512)[:views]
lib = nat.load()
lib.g6r_debug_cta_trace.restype = ctypes.c_int
lib.g6r_debug_cta_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
raster.render_views(s, cams, config=cfg, concurrency=batch)
torch.cuda.synchronize()
buf = np.zeros((1 << 17, 4), dtype=np.uint64)
lib.g6r_debug_cta_trace(buf.ctypes.data, 1 << 17)   # drop the warm-up
raster.render_views(s, cams, config=cfg, concurrency=batch, pipeline=False)
torch.cuda.synchronize()
n = lib.g6r_debug_cta_trace(buf.ctypes.data, 1 << 17)
t = buf[:n].astype(np.int64)
t0, t1 = t[:, 0], t[:, 1]
order = np.argsort(t0)
# a launch starts when a CTA starts after every earlier CTA has ended
bounds, cur, end = [], [], -1
for i in order:
    if cur and t0[i] > end:
        bounds.append(np.array(cur))
        cur = []
    cur.append(i)
    end = max(end, t1[i])
bounds.append(np.array(cur))
out = []
for k, idx in enumerate(bounds):
    a, b = t0[idx].min(), t1[idx].max()
    dur = (t1[idx] - t0[idx]) / 1e3
    top = np.argsort(-dur)[:5]
    slices = np.linspace(a, b, 21)
    # resident CTAs (time-weighted) per twentieth of the launch
    busy = []
    for j in range(20):
        lo_, hi_ = slices[j], slices[j + 1]
        ov = np.clip(np.minimum(t1[idx], hi_) - np.maximum(t0[idx], lo_), 0, None)
        busy.append(round(float(ov.sum() / (hi_ - lo_)), 1))
    out.append({"launch": k, "ctas": int(len(idx)), "span_us": (b - a) / 1e3,
                "last_start_us": (t0[idx].max() - a) / 1e3,
                "mean_cta_us": float(dur.mean()),
                "longest": [{"us": float(dur[i]), "run": int(t[idx][i, 3]),
                             "start_us": float((t0[idx][i] - a) / 1e3)} for i in top],
                "resident_ctas_per_twentieth": busy,
                "work_us_over_full_machine": float(dur.sum() / 1184.0)})
print(json.dumps(out, indent=1))
