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


def _gather_worker(rank, world, port, result_dir):
    """Served-frame gather: rank r's block of views reaches rank 0 in view order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 7   # blocks of 3 and 4 views
        mine = multigpu.shard_views(n, world, rank)
        frames = torch.stack([torch.full((5, 6, 4), v, dtype=torch.uint8) for v in mine])
        got = multigpu.gather_frames(frames, n, dst=0)
        if rank == 0:
            ok = got is not None and got.shape == (n, 5, 6, 4) and all(
                bool((got[v] == v).all()) for v in range(n))
        else:
            ok = got is None
        with open(os.path.join(result_dir, f"g{rank}"), "w") as fh:
            fh.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


def test_gather_frames_world2(tmp_path):
    world = 2
    mp.spawn(_gather_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"g{r}").read_text() == "ok"


def _dp_worker(rank, world, port, result_dir):
    """Data-parallel fine-tune host logic: the view schedule is identical on
    every rank and the bucketed gradient all-reduce averages in place."""
    from paper_2505_17338_b200 import diffrender as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sched = torch.from_numpy(D.dp_view_schedule(7, 9, 12, world))
        gathered = [torch.zeros_like(sched) for _ in range(world)]
        dist.all_gather(gathered, sched)
        ok = all(torch.equal(g, gathered[0]) for g in gathered)
        # world-1 column 0 reproduces finetune's single-rank draws
        rng = np.random.default_rng(7)
        ok = ok and [int(rng.integers(9)) for _ in range(12)] == D.dp_view_schedule(7, 9, 12, 1)[:, 0].tolist()
        grads = [torch.full((5, 3), float(rank + 1), dtype=torch.float64),
                 torch.arange(4, dtype=torch.float64) * (rank + 1)]
        D.allreduce_mean(grads)
        mean = sum(r + 1 for r in range(world)) / world
        ok = ok and torch.equal(grads[0], torch.full((5, 3), mean, dtype=torch.float64))
        ok = ok and torch.allclose(grads[1], torch.arange(4, dtype=torch.float64) * mean)
        with open(os.path.join(result_dir, f"dp{rank}"), "w") as fh:
            fh.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


def test_data_parallel_finetune_host_logic_world2(tmp_path):
    world = 2
    mp.spawn(_dp_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"dp{r}").read_text() == "ok"


def _subgroup_worker(rank, world, port, result_dir):
    """src/dst are ranks *within* the group: with group = global ranks [1, 2],
    group rank 0 is global rank 1 (the scene source and the gather target)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        group = dist.new_group([1, 2])
        ok = True
        if rank in (1, 2):
            src_scene = scenes.random_scene(np.random.default_rng(5), 64) if rank == 1 else None
            ds = multigpu.broadcast_scene(src_scene, torch.device("cpu"), src=0, group=group)
            want = scenes.random_scene(np.random.default_rng(5), 64)
            ok = np.array_equal(ds.mu_p.numpy(), want.mu_p)
            gr = dist.get_rank(group)
            mine = multigpu.shard_views(5, 2, gr)
            frames = torch.stack([torch.full((2, 3, 4), v, dtype=torch.uint8) for v in mine])
            got = multigpu.gather_frames(frames, 5, dst=0, group=group)
            if rank == 1:
                ok = ok and got is not None and all(bool((got[v] == v).all()) for v in range(5))
            else:
                ok = ok and got is None
        with open(os.path.join(result_dir, f"sg{rank}"), "w") as fh:
            fh.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


def test_broadcast_and_gather_in_a_subgroup_world3(tmp_path):
    world = 3
    mp.spawn(_subgroup_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"sg{r}").read_text() == "ok"
