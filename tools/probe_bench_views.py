"""Probe (dev tool): the bench's own timed views (cfg3, first 20 views of the
100-view orbit, balanced 10 + 10 batches) rendered once more on one stream,
so an ncu launch list / G6R_TRACE trace of this process lines up with the
bench's CUDA-event stage split.

    python tools/probe_bench_views.py [--views 20] [--batch 16] [--reps 1]
With G6R_TRACE=1 the per-launch device intervals go to gpurun_out/trace_bench.csv."""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_17338_b200 import _native as nat  # noqa: E402
from paper_2505_17338_b200 import raster  # noqa: E402
from paper_2505_17338_b200.raster import RenderConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=20)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--exp", default="fast")
a = ap.parse_args()
cfg = RenderConfig(exp_mode=a.exp)
s = bench.make_scene(bench.N_GAUSS)
lo, hi = s.mu_p.min(axis=0), s.mu_p.max(axis=0)
cams = bench.orbit_from_bbox(lo, hi, max(100, a.views), a.size)[:a.views]
prep = raster.prepare_scene(s)
_, cnt = raster.render_views(s, cams, config=cfg)
torch.cuda.synchronize()
prep.entry_hint = int(cnt[:, 1].max().item() * 1.5) + 65536
out = torch.empty((len(cams), a.size, a.size, 4), dtype=torch.float32, device="cuda")
raster.render_views(s, cams, config=cfg, out=out, concurrency=a.batch, pipeline=False)
torch.cuda.synchronize()
if os.environ.get("G6R_TRACE") == "1":
    nat.load().g6r_trace_dump(b"/tmp/g6r_trace_warm.csv")
prof = nat.Profiler(64)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    raster.render_views(s, cams, config=cfg, out=out, concurrency=a.batch, profiler=prof)
e1.record()
torch.cuda.synchronize()
stage, nv = prof.read()
res = {"views": nv, "wall_ms_per_view": e0.elapsed_time(e1) / nv,
       "stage_ms_per_view": {k: v / nv for k, v in stage.items()}}
if os.environ.get("G6R_TRACE") == "1":
    path = os.path.join(ROOT, "gpurun_out", "trace_bench.csv")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    nat.load().g6r_trace_dump(path.encode())
    agg = collections.defaultdict(list)
    for line in open(path).read().splitlines()[1:]:
        k, v = line.split(",")
        agg[k].append(float(v))
    res["trace_ms_per_view"] = {k: sum(v) / nv for k, v in agg.items()}
print(json.dumps(res))
