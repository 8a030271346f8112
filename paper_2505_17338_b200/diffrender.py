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
    g = np.ascontiguousarray(grad_image, dtype=np.float64)
    want = (int(camera.height), int(camera.width), 4)
    if g.shape != want:   # diffrender.py:417-420
        raise InvalidParameterError(
            f"grad_image shape {g.shape} does not match the rendered image {want}")
    if not g.any():   # nothing to propagate; the selection policy still applies (:414)
        cfg = replace(config, precision="f64")
        _check_config(cfg)
        _selection(prepare_scene(scene, cfg.w_mode), group_mask, cfg, RenderStats())
        return GradientBuffer.zeros(len(scene.mu_p))
    return render_backward_device(scene, camera, g, group_mask, config).to_host()


# ---------------------------------------------------------------------------
# Fine-tune loop on the device (diffrender.py:55-138, 442-585 of the reference)
# ---------------------------------------------------------------------------

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
POLY_POWER = 0.9
DEFAULT_LR_SCALE = {"mu_p": 0.1}
TRACE_FIELDS = ("iteration", "lr", "l1", "ssim_loss", "total")
DEFAULT_WEIGHTS = (0.0448, 0.2856, 0.3001, 0.2363, 0.1333)
_SHAPES = {"mu_p": (3,), "mu_d": (3,), "cov_raw": (21,), "sh": (12,), "opacity_raw": ()}


@dataclass(frozen=True)
class LossConfig:
    """lambda_l1 * L1 + lambda_ssim * (1 - MS-SSIM); weights normalised at
    construction (diffrender.py:68-97)."""

    lambda_l1: float = 0.8
    lambda_ssim: float = 0.2
    ms_ssim_scales: int = 5
    ms_ssim_weights: tuple = DEFAULT_WEIGHTS

    def __post_init__(self):
        if self.lambda_l1 < 0.0 or self.lambda_ssim < 0.0:
            raise InvalidParameterError("loss weights must be non-negative")
        if self.lambda_l1 == 0.0 and self.lambda_ssim == 0.0:
            raise InvalidParameterError("at least one loss weight must be positive")
        if self.ms_ssim_scales < 1:
            raise InvalidParameterError("ms_ssim_scales must be >= 1")
        if self.ms_ssim_scales > 5:
            raise InvalidParameterError("ms_ssim_scales above 5 are not supported on the device")
        weights = tuple(float(w) for w in self.ms_ssim_weights)
        if len(weights) != self.ms_ssim_scales:
            raise InvalidParameterError(
                f"need {self.ms_ssim_scales} ms_ssim_weights, got {len(weights)}")
        if any(w <= 0.0 for w in weights):
            raise InvalidParameterError("ms_ssim_weights must be positive")
        total = sum(weights)
        object.__setattr__(self, "ms_ssim_weights", tuple(w / total for w in weights))


class _LossWorkspace:
    """Per-(device, size) scratch for g6r_loss_grad, reused across calls."""

    _cache = {}

    @classmethod
    def get(cls, dev, w, h):
        import torch
        key = (dev.index, w, h)
        ws = cls._cache.get(key)
        if ws is None:
            nbytes = nat.load().g6r_loss_workspace_bytes(w, h)
            ws = cls._cache[key] = (torch.empty(nbytes, dtype=torch.uint8, device=dev), nbytes)
        return ws


def loss_device(pred, target, cfg: LossConfig = None, grad_out=None):
    """(total, l1, ssim_loss), grad for device tensors: pred (H,W,4) f64,
    target (H,W,3|4) f64.  One g6r_loss_grad call (synchronises the stream to
    read the three scalars)."""
    import torch
    cfg = cfg or LossConfig()
    if pred.ndim != 3 or target.ndim != 3 or tuple(pred.shape[:2]) != tuple(target.shape[:2]):
        raise InvalidParameterError(
            f"image shapes do not match: {tuple(pred.shape)} vs {tuple(target.shape)}")
    h, w = int(pred.shape[0]), int(pred.shape[1])
    if pred.shape[2] != 4 or target.shape[2] not in (3, 4):
        raise InvalidParameterError("pred must be (H,W,4) and target (H,W,3|4)")
    ws, nbytes = _LossWorkspace.get(pred.device, w, h)
    grad = grad_out if grad_out is not None else torch.empty_like(pred)
    weights = (ctypes.c_double * cfg.ms_ssim_scales)(*cfg.ms_ssim_weights)
    parts = (ctypes.c_double * 3)()
    nat.check(nat.load().g6r_loss_grad(
        _ptr(pred), _ptr(target), int(target.shape[2]), w, h, cfg.lambda_l1, cfg.lambda_ssim,
        cfg.ms_ssim_scales, ctypes.cast(weights, ctypes.c_void_p), _ptr(ws), nbytes, _ptr(grad),
        ctypes.cast(parts, ctypes.c_void_p), _stream_handle()))
    return (parts[0], parts[1], parts[2]), grad


def _to_device_image(img, dev, rgb4=False):
    import torch
    t = img if isinstance(img, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(img, np.float64))
    t = t.to(device=dev, dtype=torch.float64).contiguous()
    if t.ndim != 3:
        raise InvalidParameterError(f"expected an (H, W, C) image, got shape {tuple(t.shape)}")
    if rgb4 and t.shape[2] == 3:
        t = torch.cat([t, torch.zeros_like(t[:, :, :1])], dim=2).contiguous()
    return t


def _loss_parts(pred, gt, cfg: LossConfig):
    """(total, l1, ssim_loss, d total/d pred) comparing RGB (diffrender.py:117-138)."""
    import torch
    from .raster import _require_cuda
    _require_cuda()
    pred_a, gt_a = np.asarray(pred, np.float64), np.asarray(gt, np.float64)
    if pred_a.shape[:2] != gt_a.shape[:2] or pred_a.ndim != 3 or gt_a.ndim != 3:
        raise InvalidParameterError(f"image shapes do not match: {pred_a.shape} vs {gt_a.shape}")
    dev = torch.device("cuda", torch.cuda.current_device())
    p = _to_device_image(pred_a, dev, rgb4=True)
    g = _to_device_image(gt_a, dev)
    if g.shape[2] not in (3, 4):
        g = g[:, :, :3].contiguous()
    (total, l1, ssim_loss), grad = loss_device(p, g, cfg)
    return total, l1, ssim_loss, grad[:, :, :pred_a.shape[2]].cpu().numpy()


def loss(pred, gt, cfg: LossConfig = None):
    """Photometric loss and its analytic gradient with respect to ``pred``
    (diffrender.py:141-156): (total, grad) with grad shaped like ``pred``."""
    total, _, _, grad = _loss_parts(pred, gt, cfg or LossConfig())
    return total, grad


def ms_ssim(a, b, scales: int = 5, weights=DEFAULT_WEIGHTS) -> float:
    """Multi-scale SSIM in [-1, 1] (diffrender.py:100-114); alpha ignored.
    Single-channel images are evaluated as three identical channels."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.ndim == 2:
        a = a[:, :, None]
    if b.ndim == 2:
        b = b[:, :, None]
    if a.shape[2] == 4:
        a = a[:, :, :3]
    if b.shape[2] == 4:
        b = b[:, :, :3]
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {a.shape} vs {b.shape}")
    if min(a.shape[0], a.shape[1]) < 11:
        raise ValueError(f"images must be at least 11 px per side, got {a.shape}")
    if a.shape[2] == 1:
        a, b = np.repeat(a, 3, axis=2), np.repeat(b, 3, axis=2)
    elif a.shape[2] != 3:
        raise ValueError(f"expected 1, 3 or 4 channels, got {a.shape[2]}")
    cfg = LossConfig(lambda_l1=0.0, lambda_ssim=1.0, ms_ssim_scales=scales,
                     ms_ssim_weights=tuple(weights[:scales]))
    _, _, ssim_loss, _ = _loss_parts(np.concatenate([a, np.zeros(a.shape[:2] + (1,))], axis=2), b, cfg)
    return 1.0 - ssim_loss


def polylr(step: int, total: int, base_lr: float) -> float:
    """``base_lr * (1 - step/total) ** 0.9`` (diffrender.py:442-449)."""
    if total <= 0:
        raise InvalidParameterError(f"total must be positive, got {total}")
    if not 0 <= step <= total:
        raise InvalidParameterError(f"step {step} outside [0, {total}]")
    return base_lr * (1.0 - step / total) ** POLY_POWER


@dataclass
class OptimizerState:
    """Adam moments per parameter group plus the lr schedule (diffrender.py:452-465)."""

    m: dict
    v: dict
    step: int
    total_steps: int
    base_lr: float
    lr_scale: dict = None
    skipped: int = 0

    def __post_init__(self):
        if self.lr_scale is None:
            self.lr_scale = dict(DEFAULT_LR_SCALE)

    def lr(self) -> float:
        return polylr(self.step, self.total_steps, self.base_lr)


def init_optimizer(scene, total_steps: int, base_lr: float = 1e-3,
                   lr_scale: dict = None) -> OptimizerState:
    """Zero-moment Adam state sized for ``scene`` (diffrender.py:468-478)."""
    if total_steps <= 0:
        raise InvalidParameterError(f"total_steps must be positive, got {total_steps}")
    shapes = {name: np.shape(getattr(scene, name)) for name in PARAM_GROUPS}
    return OptimizerState(m={k: np.zeros(s) for k, s in shapes.items()},
                          v={k: np.zeros(s) for k, s in shapes.items()},
                          step=0, total_steps=total_steps, base_lr=base_lr,
                          lr_scale=dict(DEFAULT_LR_SCALE if lr_scale is None else lr_scale))


def _with_params(scene, **arrays):
    if hasattr(scene, "with_params"):
        return scene.with_params(**arrays)
    return replace(scene, **arrays)


def adam_step(state: OptimizerState, grads: GradientBuffer, scene):
    """One bias-corrected Adam update (diffrender.py:481-509) through
    g6r_adam_step; a non-finite gradient anywhere skips the update."""
    import torch
    from .raster import _require_cuda
    _require_cuda()
    if not grads.all_finite():
        state.skipped += 1
        return scene, state
    lr_now = polylr(state.step, state.total_steps, state.base_lr)
    state.step += 1
    t = state.step
    bias1 = 1.0 - ADAM_BETA1 ** t
    bias2 = 1.0 - ADAM_BETA2 ** t
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = nat.load()
    updates = {}
    for name, g in grads.groups():
        up = [torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)
              for a in (getattr(scene, name), g, state.m[name], state.v[name])]
        lr_g = lr_now * state.lr_scale.get(name, 1.0)
        nat.check(lib.g6r_adam_step(up[0].numel(), *[_ptr(a) for a in up], lr_g, bias1, bias2,
                                    _stream_handle()))
        updates[name] = up[0].cpu().numpy()
        state.m[name] = up[2].cpu().numpy()
        state.v[name] = up[3].cpu().numpy()
    return _with_params(scene, **updates), state


def write_trace(history, path) -> None:
    """Fine-tune trace rows as CSV (diffrender.py:512-517)."""
    import csv
    with open(path, "w", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=TRACE_FIELDS)
        writer.writeheader()
        writer.writerows(history)


def save_checkpoint(scene, state: OptimizerState, path) -> None:
    """G6DS scene at ``path`` plus an optimizer sidecar ``path + '.opt.npz'``
    (diffrender.py:520-531)."""
    from .sceneio import save_scene
    save_scene(scene, path)
    arrays = {f"m_{k}": state.m[k] for k in PARAM_GROUPS}
    arrays.update({f"v_{k}": state.v[k] for k in PARAM_GROUPS})
    names = sorted(state.lr_scale)
    np.savez(str(path) + ".opt.npz", step=state.step, total_steps=state.total_steps,
             base_lr=state.base_lr, skipped=state.skipped,
             lr_scale_names=np.array(names, dtype=object),
             lr_scale_values=np.array([state.lr_scale[k] for k in names]), **arrays)


def load_checkpoint(path):
    """Inverse of :func:`save_checkpoint` (diffrender.py:534-545)."""
    from .sceneio import load_scene
    scene = load_scene(path)
    with np.load(str(path) + ".opt.npz", allow_pickle=True) as z:
        state = OptimizerState(
            m={k: z[f"m_{k}"] for k in PARAM_GROUPS}, v={k: z[f"v_{k}"] for k in PARAM_GROUPS},
            step=int(z["step"]), total_steps=int(z["total_steps"]), base_lr=float(z["base_lr"]),
            skipped=int(z["skipped"]),
            lr_scale=dict(zip(z["lr_scale_names"].tolist(), z["lr_scale_values"].tolist())))
    return scene, state


class DeviceTrainer:
    """The fine-tune state resident on one GPU: the 40 raw parameters, Adam
    moments, gradients, view targets and all scratch, as device tensors.

    ``step(view)`` runs one iteration of the reference loop
    (diffrender.py:570-581) as native calls on the current stream:
    g6r_prepare -> g6r_backward_forward (f64 render, state kept) ->
    g6r_loss_grad -> g6r_backward_apply -> g6r_any_nonfinite ->
    g6r_adam_step x5.  Host synchronisation: the degenerate-policy counts,
    the overflow counter, the loss scalars and the non-finite flag."""

    def __init__(self, scene, views, loss_cfg: LossConfig = None, config: RenderConfig = None,
                 total_steps: int = 1, base_lr: float = 1e-3, lr_scale: dict = None):
        import torch
        from .raster import _require_cuda
        _require_cuda()
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.loss_cfg = loss_cfg or LossConfig()
        self.cfg = replace(config if config is not None else DEFAULT_CONFIG, precision="f64")
        if int(self.cfg.tile_size) != 16:
            raise InvalidParameterError("the backward pass supports tile_size 16")
        self.ccfg = _check_config(self.cfg)
        self.scene = scene
        self.n = n = len(scene.mu_p)

        def up(a):
            if isinstance(a, torch.Tensor):
                return a.to(device=self.dev, dtype=torch.float64).clone().contiguous()
            return torch.from_numpy(np.array(a, dtype=np.float64)).to(self.dev)

        self.params = {k: up(getattr(scene, k)) for k in PARAM_GROUPS}
        lab = scene.labels
        self.labels = (lab.to(self.dev, torch.uint8).contiguous() if isinstance(lab, torch.Tensor)
                       else torch.from_numpy(np.ascontiguousarray(lab, np.uint8)).to(self.dev))
        self.m = {k: torch.zeros_like(t) for k, t in self.params.items()}
        self.v = {k: torch.zeros_like(t) for k, t in self.params.items()}
        self.grads = {k: torch.empty((max(n, 1),) + _SHAPES[k], dtype=torch.float64,
                                     device=self.dev) for k in PARAM_GROUPS}
        self.step_count, self.total_steps, self.base_lr, self.skipped = 0, total_steps, base_lr, 0
        self.lr_scale = dict(DEFAULT_LR_SCALE if lr_scale is None else lr_scale)
        self.views = []
        for cam, target in views:
            t = _to_device_image(target, self.dev)
            if tuple(t.shape[:2]) != (int(cam.height), int(cam.width)) or t.shape[2] not in (3, 4):
                raise InvalidParameterError(
                    f"target shape {tuple(t.shape)} does not match the camera "
                    f"({int(cam.height)}, {int(cam.width)}, 3|4)")
            self.views.append((cam, t))
        ss = np.broadcast_to(np.asarray(scene.spatial_scale, np.float64), (3,))
        self.ss = (ctypes.c_double * 3)(*ss.tolist())
        self.directional_scale = float(scene.directional_scale)
        self.w_mode = _W_MODES[self.cfg.w_mode]
        self.records = torch.empty(max(n, 1) * nat.REC_DOUBLES, dtype=torch.float64, device=self.dev)
        self.flags = torch.empty(max(n, 1), dtype=torch.uint8, device=self.dev)
        self.label_counts = torch.empty(32, dtype=torch.int64, device=self.dev)
        self.counters = torch.empty(nat.NCOUNTERS, dtype=torch.int64, device=self.dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # pinned landing buffers: the per-step label counts (degenerate policy)
        # and forward counters (entry overflow) ride the loss's one read-back
        self._h_label_counts = torch.empty(32, dtype=torch.int64).pin_memory()
        self._h_counters = torch.empty(nat.NCOUNTERS, dtype=torch.int64).pin_memory()
        self.cap = max(1 << 20, 8 * n)
        self._ws = {}
        self._img = {}
        self.lib = nat.load()

    def lr(self) -> float:
        return polylr(self.step_count, self.total_steps, self.base_lr)

    def _workspace(self, w, h):
        import torch
        key = (w, h, self.cap)
        ws = self._ws.get(key)
        if ws is None:
            nbytes = self.lib.g6r_backward_workspace_bytes(self.n, w, h, 16, self.cap)
            self._ws = {}   # one live size at a time (caps only grow)
            ws = self._ws[key] = (torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.dev),
                                  nbytes)
        return ws

    def _buffers(self, w, h):
        import torch
        b = self._img.get((w, h))
        if b is None:
            b = self._img[(w, h)] = (torch.empty((h, w, 4), dtype=torch.float64, device=self.dev),
                                     torch.empty((h, w, 4), dtype=torch.float64, device=self.dev))
        return b

    def _prepare(self):
        from .raster import ScenePrep
        p = self.params
        nat.check(self.lib.g6r_prepare(
            self.n, _ptr(p["mu_p"]), _ptr(p["mu_d"]), _ptr(p["cov_raw"]), _ptr(p["sh"]),
            _ptr(p["opacity_raw"]), _ptr(self.labels), ctypes.cast(self.ss, ctypes.c_void_p),
            self.directional_scale, self.w_mode, _ptr(self.records), _ptr(self.flags),
            _ptr(self.label_counts), _stream_handle()))
        # the counts land on the host with the step's loss read-back; the
        # degenerate policy is applied then (gradients()), before any update
        self._h_label_counts.copy_(self.label_counts, non_blocking=True)
        return ScenePrep(self.records, self.flags, self._h_label_counts.numpy(), self.n,
                         self.cfg.w_mode, self.dev)

    def step(self, view_index: int) -> dict:
        """One iteration on view ``view_index``; returns lr, l1, ssim_loss, total."""
        row = self.gradients(view_index)
        self._adam(fused_check=True)
        return row

    def gradients(self, view_index: int) -> dict:
        """Forward, loss and backward on one view: fills ``self.grads`` (device)
        and returns the loss row; no parameter update."""
        cam, target = self.views[view_index]
        w, h = int(cam.width), int(cam.height)
        prep = self._prepare()
        sc = prep.scene_struct()
        camst = _camera_struct(cam)
        image, gimg = self._buffers(w, h)
        stream = _stream_handle()
        while True:
            ws, nbytes = self._workspace(w, h)
            nat.check(self.lib.g6r_backward_forward(
                ctypes.byref(sc), 0xFFFF, ctypes.byref(camst), ctypes.byref(self.ccfg), _ptr(ws),
                nbytes, self.cap, _ptr(self.counters), _ptr(image), stream))
            self._h_counters.copy_(self.counters, non_blocking=True)
            # one synchronising read-back per step: the loss scalars (the
            # counters and label counts queued above arrive with them)
            (total, l1, ssim_loss), _ = loss_device(image, target, self.loss_cfg, grad_out=gimg)
            _selection(prep, None, self.cfg, RenderStats())   # degenerate policy (raster.py:431-440)
            c = self._h_counters.numpy()
            if not c[nat.CNT_OVERFLOW]:
                break
            self.cap = min(int(c[nat.CNT_ENTRIES] * 1.25) + 4096, (1 << 30) - 1)
        lr_now = self.lr()
        p, g = self.params, self.grads
        nat.check(self.lib.g6r_backward_apply(
            ctypes.byref(sc), ctypes.byref(camst), ctypes.byref(self.ccfg), _ptr(ws), nbytes,
            self.cap, _ptr(p["mu_p"]), _ptr(p["mu_d"]), _ptr(p["cov_raw"]), _ptr(p["sh"]),
            ctypes.cast(self.ss, ctypes.c_void_p), self.directional_scale, self.w_mode,
            _ptr(gimg), *[_ptr(g[k]) for k in PARAM_GROUPS], _ptr(self.counters), stream))
        return {"lr": lr_now, "l1": l1, "ssim_loss": ssim_loss, "total": total}

    def apply_gradients(self):
        """Adam on ``self.grads`` (skipped when any is non-finite)."""
        self._adam()

    def _adam(self, fused_check: bool = False):
        stream = _stream_handle()
        if fused_check:   # the backward flagged non-finite gradients as it wrote them
            bad = int(self.counters[nat.CNT_GRAD_NONFINITE].item())
        else:             # gradients changed since (e.g. all-reduced): check them
            self.flag.zero_()
            for k in PARAM_GROUPS:
                nat.check(self.lib.g6r_any_nonfinite(self.params[k].numel(), _ptr(self.grads[k]),
                                                     _ptr(self.flag), stream))
            bad = int(self.flag.item())
        if bad:
            self.skipped += 1
            return
        lr_now = self.lr()
        self.step_count += 1
        t = self.step_count
        bias1 = 1.0 - ADAM_BETA1 ** t
        bias2 = 1.0 - ADAM_BETA2 ** t
        for k in PARAM_GROUPS:
            nat.check(self.lib.g6r_adam_step(
                self.params[k].numel(), _ptr(self.params[k]), _ptr(self.grads[k]), _ptr(self.m[k]),
                _ptr(self.v[k]), lr_now * self.lr_scale.get(k, 1.0), bias1, bias2, stream))

    def result_scene(self):
        """The optimised parameters as a host scene of the input's type."""
        arrays = {k: t.cpu().numpy() for k, t in self.params.items()}
        if not isinstance(self.scene.mu_p, np.ndarray):
            from .multigpu import DeviceScene
            s = self.scene
            return DeviceScene(labels=s.labels, spatial_scale=s.spatial_scale,
                               directional_scale=s.directional_scale,
                               **{k: t.clone() for k, t in self.params.items()})
        return _with_params(self.scene, **arrays)

    def optimizer_state(self) -> OptimizerState:
        return OptimizerState(m={k: t.cpu().numpy() for k, t in self.m.items()},
                              v={k: t.cpu().numpy() for k, t in self.v.items()},
                              step=self.step_count, total_steps=self.total_steps,
                              base_lr=self.base_lr, lr_scale=dict(self.lr_scale),
                              skipped=self.skipped)


def finetune(scene, views, iters: int = 300, loss_cfg: LossConfig = None,
             config: RenderConfig = None, seed: int = 0, base_lr: float = 1e-3,
             lr_scale: dict = None, trace_path=None, checkpoint_path=None):
    """Optimise every per-Gaussian parameter against ``views`` on the GPU
    (diffrender.py:548-585): each iteration samples one (camera, target) pair
    with ``default_rng(seed)``, renders in f64, backpropagates the photometric
    loss and applies one Adam step under polynomial lr decay.  Returns
    ``(scene, history)``; history rows carry iteration, lr, l1, ssim_loss and
    total.  Deterministic: repeated runs are bit-identical."""
    if len(views) == 0:
        raise InvalidParameterError("finetune needs at least one view")
    if iters < 0:
        raise InvalidParameterError(f"iters must be non-negative, got {iters}")
    if iters == 0:   # the reference returns its input scene object untouched (:571-585)
        if trace_path is not None:
            write_trace([], trace_path)
        if checkpoint_path is not None:
            save_checkpoint(scene, init_optimizer(scene, 1, base_lr, lr_scale), checkpoint_path)
        return scene, []
    tr = DeviceTrainer(scene, views, loss_cfg, config, total_steps=max(iters, 1),
                       base_lr=base_lr, lr_scale=lr_scale)
    rng = np.random.default_rng(seed)
    history = []
    for it in range(iters):
        row = tr.step(int(rng.integers(len(views))))
        history.append({"iteration": it, **row})
    out = tr.result_scene()
    if trace_path is not None:
        write_trace(history, trace_path)
    if checkpoint_path is not None:
        save_checkpoint(out, tr.optimizer_state(), checkpoint_path)
    return out, history


# ---------------------------------------------------------------------------
# Data-parallel fine-tuning (SURVEY.md 8e "Fine-tune (next)")
# ---------------------------------------------------------------------------

def dp_view_schedule(seed: int, n_views: int, iters: int, world: int) -> np.ndarray:
    """(iters, world) view indices: iteration t's draws for ranks 0..world-1,
    from one ``default_rng(seed)`` stream (world = 1 reproduces ``finetune``)."""
    rng = np.random.default_rng(seed)
    return np.array([[int(rng.integers(n_views)) for _ in range(world)] for _ in range(iters)],
                    dtype=np.int64).reshape(iters, world)


def allreduce_mean(tensors, group=None):
    """Average same-dtype tensors across ranks with ONE collective: flatten into
    a bucket, all-reduce (sum), scale by 1/world, scatter back in place."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    flat.mul_(1.0 / world)
    k = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[k:k + n].view_as(t))
        k += n


def finetune_data_parallel(scene, views, iters: int = 300, loss_cfg: LossConfig = None,
                           config: RenderConfig = None, seed: int = 0, base_lr: float = 1e-3,
                           lr_scale: dict = None, group=None):
    """Data-parallel fine-tuning, one process per GPU (torch.distributed, NCCL
    over NVLink on B200 nodes): every iteration each rank renders and
    backpropagates its own view (``dp_view_schedule``), the 40-parameter
    gradients are averaged with one bucketed all-reduce, and every rank applies
    the identical Adam step, so parameters stay bit-identical across ranks.
    With one rank this is ``finetune`` exactly.  Returns ``(scene, history)``
    on every rank; history losses are averaged over ranks."""
    import torch
    import torch.distributed as dist
    if len(views) == 0:
        raise InvalidParameterError("finetune needs at least one view")
    if iters < 0:
        raise InvalidParameterError(f"iters must be non-negative, got {iters}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    tr = DeviceTrainer(scene, views, loss_cfg, config, total_steps=max(iters, 1),
                       base_lr=base_lr, lr_scale=lr_scale)
    sched = dp_view_schedule(seed, len(views), iters, world)
    history = []
    for it in range(iters):
        row = tr.gradients(int(sched[it, rank]))
        if world > 1:
            allreduce_mean([tr.grads[k][:tr.n] for k in PARAM_GROUPS], group)
            losses = torch.tensor([row["l1"], row["ssim_loss"], row["total"]], dtype=torch.float64,
                                  device=tr.dev)
            dist.all_reduce(losses, group=group)
            l1, ssim_loss, total = (losses / world).tolist()
            row = {"lr": row["lr"], "l1": l1, "ssim_loss": ssim_loss, "total": total}
        tr.apply_gradients()
        history.append({"iteration": it, **row})
    return tr.result_scene(), history
