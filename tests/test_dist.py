"""Multi-process view sharding on CPU (gloo, world size 2).

The GPU path uses the same code with backend "nccl"; here every rank checks
that the one-time scene broadcast delivers bit-identical parameters and that
the orbit blocks partition the views."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_17338_b200 import multigpu, scenes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        src_scene = scenes.random_scene(np.random.default_rng(11), 257) if rank == 0 else None
        ds = multigpu.broadcast_scene(src_scene, torch.device("cpu"), src=0)
        want = scenes.random_scene(np.random.default_rng(11), 257)
        ok = all(np.array_equal(getattr(ds, f).numpy(), getattr(want, f))
                 for f in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"))
        ok = ok and np.array_equal(ds.spatial_scale, want.spatial_scale)
        mine = multigpu.shard_views(100, world, rank)
        counts = torch.tensor([len(mine), mine.start], dtype=torch.int64)
        gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, counts)
        total = sum(int(g[0]) for g in gathered)
        starts = sorted(int(g[1]) for g in gathered)
        ok = ok and total == 100 and starts == [0, 50]
        with open(os.path.join(result_dir, f"rank{rank}"), "w") as fh:
            fh.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


def test_broadcast_and_shard_world2(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"rank{r}").read_text() == "ok"
