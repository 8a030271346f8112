"""Probe: device time of each fine-tune phase (forward with state, loss +
image gradient, backward, Adam), each bracketed by CUDA events with a sync,
against the free-running iteration time (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_17338_b200 import diffrender as D, scenes

scene = scenes.psi_decode_scene()
cams = scenes.orbit_ring(scene, count=8, size=512)
views = [(c, scenes.synthetic_target(512, 512, seed=k)) for k, c in enumerate(cams)]
tr = D.DeviceTrainer(scene, views, total_steps=1000)
for k in range(3):
    tr.step(k)
torch.cuda.synchronize()
orig = {name: getattr(tr.lib, name) for name in ("g6r_backward_forward", "g6r_loss_grad",
                                                  "g6r_backward_apply", "g6r_adam_step",
                                                  "g6r_any_nonfinite")}
acc = {k: 0.0 for k in orig}


def wrap(name):
    f = orig[name]

    def g(*a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = f(*a)
        e1.record()
        torch.cuda.synchronize()
        acc[name] += e0.elapsed_time(e1)
        return r
    return g


iters = 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(iters):
    tr.step(k % 8)
e1.record()
torch.cuda.synchronize()
free = e0.elapsed_time(e1) / iters
for name in orig:
    setattr(tr.lib, name, wrap(name))
for k in range(iters):
    tr.step(k % 8)
print(f"free-running {free:.3f} ms/iter; phases (ms/iter):",
      {k.replace("g6r_", ""): round(v / iters, 3) for k, v in acc.items()},
      "sum", round(sum(acc.values()) / iters, 3))
