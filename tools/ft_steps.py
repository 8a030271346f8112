"""Run a few DeviceTrainer steps on the bench's 1M-Gaussian scene (dev tool;
the subject of the fine-tune launch list, tools/ft_step_table.py):
    python tools/ft_steps.py [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17338_b200 import diffrender as D, scenes
scene = scenes.psi_decode_scene()
cams = scenes.orbit_ring(scene, count=8, size=512)
views = [(c, scenes.synthetic_target(512, 512, seed=k)) for k, c in enumerate(cams)]
tr = D.DeviceTrainer(scene, views, total_steps=1000)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6): tr.step(k % 8)
torch.cuda.synchronize()
print("ok")
