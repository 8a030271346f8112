"""Scene ingest on the device.

* ``decode_param_volume_device``: the 37-channel parameter volume Psi on the
  half-resolution grid -> a device-resident scene (priming.py:232-285), as one
  count + scan + emit stream compaction over the half-grid voxels
  (g6r_decode_param_volume*).  ``decode_param_volume`` returns the same rows as
  a host ``Scene`` (the reference's signature).
* ``filter_scene_device``: group subset of a device scene, order kept
  (priming.py:362-374), by the same compaction (g6r_filter_rows).
* ``load_param_volume`` / ``save_param_volume``: the .meta/.raw pair
  (priming.py:314-359); the f32 payload is kept as f32 and widened on the
  device.

Accepts the reference's own ``ParamVolume`` / ``InputVolume6`` /
``LabelVolume`` objects (duck-typed on ``channels``, ``labels``,
``consolidated``, ``spacing``, ``origin``, ``direction``).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _native as nat
from .errors import EmptySceneError, InvalidParameterError, VolumeFormatError
from .scene import N_GROUPS

N_PSI_CHANNELS = 37


class ParamVolume:
    """37-channel per-voxel Gaussian parameters at half input resolution;
    channels (37, D', H', W') f32 or f64, finite."""

    def __init__(self, channels):
        data = np.asarray(channels)
        if data.dtype not in (np.float32, np.float64):
            data = data.astype(np.float64)
        if data.ndim != 4 or data.shape[0] != N_PSI_CHANNELS:
            raise InvalidParameterError(
                f"channels must have shape (37, D', H', W'), got {data.shape}")
        if not np.all(np.isfinite(data)):
            raise InvalidParameterError("channels contain non-finite values")
        self.channels = data

    @property
    def dims(self):
        return tuple(self.channels.shape[1:])


def load_param_volume(path) -> ParamVolume:
    """Read ``<path>.meta`` + ``<path>.raw`` (channel-major little-endian f32)."""
    path = Path(path)
    meta, raw = path.with_suffix(".meta"), path.with_suffix(".raw")
    if not meta.is_file():
        raise VolumeFormatError(f"missing descriptor {meta}")
    if not raw.is_file():
        raise VolumeFormatError(f"missing payload {raw}")
    kv = {}
    for line in meta.read_text(encoding="utf-8").splitlines():
        line = line.strip()
        if line and not line.startswith("#"):
            k, _, v = line.partition("=")
            kv[k.strip()] = v.strip()
    try:
        channels = int(kv["channels"])
        dims = tuple(int(x) for x in kv["dims"].split())
    except (KeyError, ValueError) as exc:
        raise VolumeFormatError(f"{meta}: bad descriptor: {exc}") from exc
    if channels != N_PSI_CHANNELS or len(dims) != 3:
        raise VolumeFormatError(f"{meta}: expected 37 channels and 3 dims, got {channels} "
                                f"channels, dims {dims}")
    payload = raw.read_bytes()
    want = channels * dims[0] * dims[1] * dims[2] * 4
    if len(payload) != want:
        raise VolumeFormatError(f"{raw}: payload is {len(payload)} bytes, descriptor implies {want}")
    return ParamVolume(np.frombuffer(payload, dtype="<f4").reshape((channels,) + dims))


def save_param_volume(psi: ParamVolume, path) -> None:
    path = Path(path)
    d = psi.dims
    path.with_suffix(".meta").write_text(f"channels={N_PSI_CHANNELS}\ndims={d[0]} {d[1]} {d[2]}\n",
                                         encoding="utf-8")
    path.with_suffix(".raw").write_bytes(np.asarray(psi.channels).astype("<f4").tobytes())


def _half_grid_inputs(psi, in6, labels):
    """Validation of priming.py:248-258 and the half-grid views (:225-229)."""
    if not labels.consolidated:
        raise InvalidParameterError("labels must be consolidated")
    lab_full = np.asarray(labels.labels)
    ch = np.asarray(in6.channels)
    if tuple(lab_full.shape) != tuple(ch.shape[1:]):
        raise VolumeFormatError(
            f"labels dims {tuple(lab_full.shape)} do not match volume dims {tuple(ch.shape[1:])}")
    expected = tuple(d // 2 for d in ch.shape[1:])
    pdims = tuple(np.shape(psi.channels)[1:])
    if pdims != expected or min(expected) < 1:
        raise VolumeFormatError(
            f"parameter volume dims {pdims} do not match half-resolution grid {expected}")
    dp, hp, wp = expected
    lab = np.ascontiguousarray(lab_full[::2, ::2, ::2][:dp, :hp, :wp], dtype=np.uint8)
    base = np.ascontiguousarray(ch[2:6, ::2, ::2, ::2][:, :dp, :hp, :wp], dtype=np.float64)
    return expected, lab, base


def decode_param_volume_device(psi, in6, labels, device=None):
    """Decode Psi into a device-resident scene (``multigpu.DeviceScene``)."""
    import torch

    from .multigpu import DeviceScene
    from .raster import _ptr, _require_cuda, _stream_handle

    _require_cuda()
    dims, lab, base = _half_grid_inputs(psi, in6, labels)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    chans = psi.channels
    f32 = isinstance(chans, np.ndarray) and chans.dtype == np.float32
    lib = nat.load()
    V = int(np.prod(dims))
    with torch.cuda.device(dev):
        host = np.ascontiguousarray(chans)
        psi_t = torch.from_numpy(host if host.flags.writeable else host.copy()).to(dev)
        lab_t = torch.from_numpy(lab).to(dev)
        base_t = torch.from_numpy(base).to(dev)
        nbytes = lib.g6r_compact_workspace_bytes(V)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        d = (ctypes.c_int32 * 3)(*dims)
        nat.check(lib.g6r_decode_param_volume_count(d, _ptr(lab_t), _ptr(ws), nbytes, _ptr(count),
                                                    _stream_handle()))
        n = int(count.item())
        if n == 0:
            raise EmptySceneError("half-resolution grid has no foreground voxels")
        out = [torch.empty((n,) + s, dtype=torch.float64, device=dev)
               for s in ((3,), (3,), (21,), (12,), ())]
        labels_t = torch.empty(n, dtype=torch.uint8, device=dev)
        sp = np.ascontiguousarray(in6.spacing, np.float64)
        og = np.ascontiguousarray(in6.origin, np.float64)
        dr = np.ascontiguousarray(in6.direction, np.float64)
        nat.check(lib.g6r_decode_param_volume(
            d, _ptr(psi_t), int(f32), _ptr(base_t), _ptr(lab_t),
            sp.ctypes.data_as(ctypes.c_void_p), og.ctypes.data_as(ctypes.c_void_p),
            dr.ctypes.data_as(ctypes.c_void_p), _ptr(ws), nbytes, *[_ptr(t) for t in out],
            _ptr(labels_t), _stream_handle()))
    mu_p, mu_d, cov_raw, sh, opacity_raw = out
    return DeviceScene(mu_p=mu_p, mu_d=mu_d, cov_raw=cov_raw, sh=sh, opacity_raw=opacity_raw,
                       labels=labels_t, spatial_scale=np.asarray(in6.spacing, np.float64),
                       directional_scale=1.0, spacing=in6.spacing, origin=in6.origin,
                       direction=in6.direction)


def decode_param_volume(psi, in6, labels):
    """Host ``Scene`` from Psi (priming.py:232-285), computed on the device."""
    return decode_param_volume_device(psi, in6, labels).to_host()


def filter_scene_device(scene, group_mask):
    """Rows of a device scene whose label is in ``group_mask`` (iterable of
    ints), order kept (priming.py:362-374)."""
    import torch

    from .multigpu import DeviceScene
    from .raster import _ptr, _require_cuda, _stream_handle

    _require_cuda()
    bits = 0
    for g in group_mask:
        if not 0 <= int(g) < N_GROUPS:
            raise InvalidParameterError(f"group index {g} outside [0, 11]")
        bits |= 1 << int(g)
    n = len(scene)
    dev = scene.mu_p.device
    lib = nat.load()
    with torch.cuda.device(dev):
        nbytes = lib.g6r_compact_workspace_bytes(n)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        out = [torch.empty((max(n, 1),) + s, dtype=torch.float64, device=dev)
               for s in ((3,), (3,), (21,), (12,), ())]
        labels = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        src = [scene.mu_p, scene.mu_d, scene.cov_raw, scene.sh, scene.opacity_raw]
        src = [t.contiguous() for t in src]
        nat.check(lib.g6r_filter_rows(n, _ptr(scene.labels.contiguous()), bits,
                                      *[_ptr(t) for t in src], _ptr(ws), nbytes,
                                      *[_ptr(t) for t in out], _ptr(labels), _ptr(count),
                                      _stream_handle()))
        m = int(count.item())
    mu_p, mu_d, cov_raw, sh, opacity_raw = (t[:m] for t in out)
    return DeviceScene(mu_p=mu_p, mu_d=mu_d, cov_raw=cov_raw, sh=sh, opacity_raw=opacity_raw,
                       labels=labels[:m], spatial_scale=scene.spatial_scale,
                       directional_scale=scene.directional_scale,
                       spacing=getattr(scene, "spacing", None), origin=getattr(scene, "origin", None),
                       direction=getattr(scene, "direction", None))
