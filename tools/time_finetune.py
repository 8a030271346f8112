"""Time the on-device fine-tune loop (BASELINE.json configs[4]).

1M-Gaussian psi_decode_scene, 512x512 orbit views with synthetic targets,
``iters`` iterations of diffrender.DeviceTrainer.step; prints per-iteration
device time (CUDA events) and the phase split.  Usage:
    python tools/time_finetune.py [--iters 30] [--views 8] [--size 512]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_17338_b200 import diffrender as D  # noqa: E402
from paper_2505_17338_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--limit", type=int, default=None)
    a = ap.parse_args()
    t0 = time.time()
    scene = scenes.psi_decode_scene(limit=a.limit)
    cams = scenes.orbit_ring(scene, count=a.views, size=a.size)
    views = [(c, scenes.synthetic_target(a.size, a.size, seed=k)) for k, c in enumerate(cams)]
    t_build = time.time() - t0
    tr = D.DeviceTrainer(scene, views, total_steps=max(300, a.iters + 3))
    rng = np.random.default_rng(0)
    for _ in range(3):
        tr.step(int(rng.integers(len(views))))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    w0 = time.perf_counter()
    rows = [tr.step(int(rng.integers(len(views)))) for _ in range(a.iters)]
    ev[1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    ms = ev[0].elapsed_time(ev[1]) / a.iters
    print(json.dumps({"n": len(scene.mu_p), "size": a.size, "iters": a.iters,
                      "ms_per_iter_device": ms, "ms_per_iter_wall": 1e3 * wall / a.iters,
                      "projected_300_iters_s": 0.3 * ms, "scene_build_s": t_build,
                      "last": rows[-1]}))


if __name__ == "__main__":
    main()
