"""View-parallel rendering across GPUs (one process per GPU).

The render path shards naturally over camera views: once the
Gaussian set is resident, views are independent.  So the only collective is a
one-time broadcast of the scene's parameter SoA from the source rank
(``torch.distributed`` with backend ``nccl`` over NVLink on B200 nodes,
``gloo`` for CPU tests); each rank then prepares the scene locally and renders
the contiguous block ``[g*V/G, (g+1)*V/G)`` of the orbit.  There is no
per-view exchange and no data-path collective.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

# column layout of the packed broadcast payload (float64, N x 40)
_COLS = (("mu_p", 3), ("mu_d", 3), ("cov_raw", 21), ("sh", 12), ("opacity_raw", 1))
N_PARAMS = 40


class DeviceScene:
    """Scene whose parameter arrays already live on a device (torch tensors).

    Accepted wherever the renderer takes a scene: ``prepare_scene`` uploads
    nothing and prepares straight from these tensors."""

    def __init__(self, mu_p, mu_d, cov_raw, sh, opacity_raw, labels, spatial_scale,
                 directional_scale, spacing=None, origin=None, direction=None):
        self.mu_p = mu_p
        self.mu_d = mu_d
        self.cov_raw = cov_raw
        self.sh = sh
        self.opacity_raw = opacity_raw
        self.labels = labels
        self.spatial_scale = np.asarray(spatial_scale, dtype=np.float64)
        self.directional_scale = float(directional_scale)
        self.spacing = np.ones(3) if spacing is None else np.asarray(spacing, np.float64)
        self.origin = np.zeros(3) if origin is None else np.asarray(origin, np.float64)
        self.direction = np.eye(3) if direction is None else np.asarray(direction, np.float64)

    def __len__(self):
        return int(self.mu_p.shape[0])

    def to_host(self):
        """Host ``Scene`` with the same parameters (one D2H copy per array)."""
        from .scene import Scene
        return Scene(mu_p=self.mu_p.cpu().numpy(), mu_d=self.mu_d.cpu().numpy(),
                     cov_raw=self.cov_raw.cpu().numpy(), sh=self.sh.cpu().numpy(),
                     opacity_raw=self.opacity_raw.cpu().numpy(), labels=self.labels.cpu().numpy(),
                     spacing=self.spacing, origin=self.origin, direction=self.direction,
                     spatial_scale=self.spatial_scale, directional_scale=self.directional_scale)


def shard_views(n_views: int, world: int, rank: int) -> range:
    """Contiguous block of views owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return range(rank * n_views // world, (rank + 1) * n_views // world)


def pack_scene(scene, device) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(N,40) float64 params, (N,) uint8 labels, (4,) float64 scales."""
    params = np.concatenate([np.asarray(getattr(scene, name), dtype=np.float64).reshape(-1, w)
                             for name, w in _COLS], axis=1)
    scales = np.concatenate([np.broadcast_to(np.asarray(scene.spatial_scale, np.float64), (3,)),
                             [float(scene.directional_scale)]])
    return (torch.from_numpy(np.ascontiguousarray(params)).to(device),
            torch.from_numpy(np.ascontiguousarray(scene.labels, dtype=np.uint8)).to(device),
            torch.from_numpy(scales).to(device))


def unpack_scene(params: torch.Tensor, labels: torch.Tensor, scales: torch.Tensor) -> DeviceScene:
    cols, k = {}, 0
    for name, w in _COLS:
        t = params[:, k:k + w]
        cols[name] = t.reshape(-1).contiguous() if w == 1 else t.contiguous()
        k += w
    sc = scales.cpu().numpy()
    return DeviceScene(spatial_scale=sc[:3], directional_scale=sc[3], labels=labels.contiguous(),
                       **cols)


def _staged(t: torch.Tensor, group) -> torch.Tensor:
    """gloo moves host tensors only for some collectives: stage device tensors
    through host memory there (NCCL takes device tensors directly)."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu()
    return t


def broadcast_scene(scene, device, src: int = 0, group=None) -> DeviceScene:
    """Broadcast ``scene`` (given on rank ``src`` of ``group``, ignored
    elsewhere) to every rank of ``group``; ``src`` is a rank *within* the
    group (the default group: the global rank).

    Three collectives in total per scene: the row count, the (N,40) float64
    parameters plus the label bytes, and the 4 scales."""
    rank = dist.get_rank(group)
    n = torch.zeros(1, dtype=torch.int64, device=device)
    if rank == src:
        n[0] = len(scene.mu_p)
    n = _bcast(n, src, group)
    n = int(n.item())
    if rank == src:
        params, labels, scales = pack_scene(scene, device)
    else:
        params = torch.empty((n, N_PARAMS), dtype=torch.float64, device=device)
        labels = torch.empty(n, dtype=torch.uint8, device=device)
        scales = torch.empty(4, dtype=torch.float64, device=device)
    params = _bcast(params, src, group)
    labels = _bcast(labels, src, group)
    scales = _bcast(scales, src, group)
    return unpack_scene(params, labels, scales)


def _bcast(t: torch.Tensor, src: int, group) -> torch.Tensor:
    s = _staged(t, group)
    dist.broadcast(s, group=group, group_src=src)
    if s is not t:
        t.copy_(s)
    return t


def gather_frames(frames: torch.Tensor, n_views: int, dst: int = 0, group=None):
    """Collect every rank's block of served frames on ``dst`` (SURVEY.md 8e,
    "optionally gather uint8 frames to rank 0"); ``dst`` is a rank within
    ``group``.

    ``frames`` holds this rank's ``shard_views`` block, (V_r, H, W, 4) on its
    device (the blocks differ in length by at most one).  Each rank sends one
    block padded to ceil(n_views / world) views through a single gather; rank
    ``dst`` returns the (n_views, H, W, 4) frames in view order, the others
    None.  Not part of the view-parallel render itself (no data-path
    collective); the bench times it separately."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard_views(n_views, world, rank)
    if frames.shape[0] != len(mine):
        raise ValueError(f"rank {rank} holds {frames.shape[0]} frames, its block has {len(mine)}")
    per = -(-n_views // world)
    buf = torch.zeros((per,) + tuple(frames.shape[1:]), dtype=frames.dtype, device=frames.device)
    buf[:len(mine)] = frames
    buf = _staged(buf, group)
    out = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, out, group=group, group_dst=dst)
    if rank != dst:
        return None
    return torch.cat([out[r][:len(shard_views(n_views, world, r))] for r in range(world)])
