"""Backward render on the B200: analytic gradients of the render path.

Mirrors the reference's ``splatct.diffrender.render_backward`` /
``GradientBuffer`` (diffrender.py:159-180, 401-439): given d loss / d image
for one view, returns the loss partials of all 40 raw parameters of every
Gaussian.  Runs as one call into ``g6r_render_backward`` (include/g6r.h): an
f64 forward of the view, the adjoint compositor, a deterministic per-splat
reduction and the chain through conic, EWA Jacobian, camera, slicing,
covariance, Cholesky factor, SH and sigmoid.  Culled, masked and degenerate
Gaussians receive exact zeros, as in the reference.  No CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from .errors import InvalidParameterError
from .raster import (DEFAULT_CONFIG, RenderConfig, RenderStats, _camera_struct, _check_config,
                     _ptr, _selection, _stream_handle, _W_MODES, prepare_scene)

PARAM_GROUPS = ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw")   # diffrender.py:63


@dataclass
class GradientBuffer:
    """Loss partials for every per-Gaussian parameter, row-aligned with a scene."""

    mu_p: np.ndarray
    mu_d: np.ndarray
    cov_raw: np.ndarray
    sh: np.ndarray
    opacity_raw: np.ndarray

    @classmethod
    def zeros(cls, n: int) -> "GradientBuffer":
        return cls(mu_p=np.zeros((n, 3)), mu_d=np.zeros((n, 3)), cov_raw=np.zeros((n, 21)),
                   sh=np.zeros((n, 12)), opacity_raw=np.zeros(n))

    def groups(self):
        return tuple((name, getattr(self, name)) for name in PARAM_GROUPS)

    def all_finite(self) -> bool:
        return all(np.all(np.isfinite(arr)) for _, arr in self.groups())


class DeviceGradients:
    """The five gradient arrays as device tensors (no host transfer)."""

    def __init__(self, mu_p, mu_d, cov_raw, sh, opacity_raw, image, counters):
        self.mu_p, self.mu_d, self.cov_raw, self.sh, self.opacity_raw = mu_p, mu_d, cov_raw, sh, opacity_raw
        self.image = image
        self.counters = counters

    def to_host(self) -> GradientBuffer:
        return GradientBuffer(self.mu_p.cpu().numpy(), self.mu_d.cpu().numpy(),
                              self.cov_raw.cpu().numpy(), self.sh.cpu().numpy(),
                              self.opacity_raw.cpu().numpy())


def render_backward_device(scene, camera, grad_image, group_mask=None,
                           config: RenderConfig = DEFAULT_CONFIG) -> DeviceGradients:
    """Device-resident variant: ``grad_image`` may be a CUDA tensor or array."""
    import torch
    from .raster import _device_scene

    cfg = replace(config, precision="f64")
    if int(cfg.tile_size) != 16:
        raise InvalidParameterError("the backward pass supports tile_size 16")
    ccfg = _check_config(cfg)
    prep = prepare_scene(scene, cfg.w_mode)
    bits = _selection(prep, group_mask, cfg, RenderStats())
    ds = _device_scene(scene)
    dev = prep.device
    H, W = int(camera.height), int(camera.width)
    if isinstance(grad_image, torch.Tensor):
        g = grad_image.to(device=dev, dtype=torch.float64).contiguous()
    else:
        g = torch.from_numpy(np.ascontiguousarray(grad_image, dtype=np.float64)).to(dev)
    if tuple(g.shape) != (H, W, 4):
        raise InvalidParameterError(
            f"grad_image shape {tuple(g.shape)} does not match the rendered image {(H, W, 4)}")
    n = prep.n
    cam = _camera_struct(camera)
    sc = prep.scene_struct()
    ss = (ctypes.c_double * 3)(*ds.spatial_scale.tolist())
    lib = nat.load()
    while True:
        cap = int(prep.entry_hint)
        nbytes = lib.g6r_backward_workspace_bytes(n, W, H, 16, cap)
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        out = [torch.empty((max(n, 1),) + s, dtype=torch.float64, device=dev)
               for s in ((3,), (3,), (21,), (12,), ())]
        image = torch.empty((H, W, 4), dtype=torch.float64, device=dev)
        counters = torch.empty(nat.NCOUNTERS, dtype=torch.int64, device=dev)
        nat.check(lib.g6r_render_backward(
            ctypes.byref(sc), bits, ctypes.byref(cam), ctypes.byref(ccfg), _ptr(ws), nbytes, cap,
            _ptr(ds.mu_p), _ptr(ds.mu_d), _ptr(ds.cov_raw), _ptr(ds.sh),
            ctypes.cast(ss, ctypes.c_void_p), ds.directional_scale, _W_MODES[cfg.w_mode], _ptr(g),
            *[_ptr(t) for t in out], _ptr(counters), _ptr(image), _stream_handle()))
        c = counters.cpu().numpy()
        if not c[nat.CNT_OVERFLOW]:
            break
        prep.entry_hint = min(int(c[nat.CNT_ENTRIES] * 1.25) + 4096, (1 << 30) - 1)
    return DeviceGradients(*[t[:n] for t in out], image, counters)


def render_backward(scene, camera, grad_image, group_mask=None,
                    config: RenderConfig = DEFAULT_CONFIG, state=None) -> GradientBuffer:
    """Loss partials for every Gaussian parameter, given d loss / d image
    (diffrender.py:401-439).  ``state`` is accepted for signature parity; the
    f64 forward is recomputed on the device (it is a small part of the cost)."""
    if config.w_mode not in _W_MODES:
        raise ValueError(f"unknown opacity modulation mode {config.w_mode!r}")
    g = np.asarray(grad_image, dtype=np.float64)
    if not g.any():
        return GradientBuffer.zeros(len(scene.mu_p))
    return render_backward_device(scene, camera, g, group_mask, config).to_host()
