"""The view-parallel multi-GPU path, exercised on ONE device.

Only one GPU is available to the tests, so two ranks share cuda:0 over the
gloo backend: the same code the NCCL run executes (scene broadcast from rank 0,
per-rank prepare, contiguous shard of the orbit, served-frame gather on rank 0)
minus the transport.  The ranks never wait on each other inside a kernel --
views are independent -- so sharing a device is safe.

1. ``multigpu`` + ``raster.render_frames_u8`` on the 1M-Gaussian benchmark
   scene: rank 0's gathered frames are byte-identical to a single-process
   render of the same views.
2. ``bench.py --gpus 2`` under torchrun with ``--dist-backend gloo`` runs end
   to end and prints one JSON line with n_gpus 2 (no scaling number: both
   ranks share a GPU)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, n_gauss, n_views, size):
    sys.path.insert(0, ROOT)
    from paper_2505_17338_b200 import multigpu, raster, scenes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        host = scenes.psi_decode_scene(352, limit=n_gauss) if rank == 0 else None
        scene = multigpu.broadcast_scene(host, dev, src=0)
        lo = scene.mu_p.amin(0).cpu().numpy()
        hi = scene.mu_p.amax(0).cpu().numpy()
        import bench
        cams = bench.orbit_from_bbox(lo, hi, n_views, size)
        mine = multigpu.shard_views(n_views, world, rank)
        frames = raster.render_frames_u8(scene, [cams[v] for v in mine], device_out=True)
        got = multigpu.gather_frames(frames, n_views, dst=0)
        if rank == 0:
            # single-process reference: the host scene, every view, one rank
            want = raster.render_frames_u8(host, cams)
            np.save(os.path.join(out_dir, "got.npy"), got.cpu().numpy())
            np.save(os.path.join(out_dir, "want.npy"), want)
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_process(tmp_path):
    world, n_views = 2, 9
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), 1_000_000, n_views, 512),
             nprocs=world, join=True)
    got = np.load(tmp_path / "got.npy")
    want = np.load(tmp_path / "want.npy")
    assert got.shape == (n_views, 512, 512, 4) and got.dtype == np.uint8
    np.testing.assert_array_equal(got, want)
    assert (got[..., :3] > 0).mean() > 0.05   # the frames show the scene


def test_bench_two_ranks_gloo_on_one_device():
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "6", "--warmup", "3",
           "--dist-backend", "gloo", "--gaussians", "200000", "--size", "256"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["unit"] == "views/s"
    assert rec["config"]["parallelism"].startswith("view-parallel x2")
    assert rec["frame_gather"].get("views") == 12
