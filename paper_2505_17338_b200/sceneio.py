"""G6DS scene files (the reference's sceneio.py format, read and written here).

Format (little-endian), as specified by the reference (sceneio.py:1-13):
``b"G6DS"``, u32 version (1), u64 count; a 152-byte metadata block (spacing 3,
origin 3, direction 3x3, spatial_scale 3, directional_scale: all f64); then
``count`` 168-byte records of f32 mu_p[3] mu_d[3] cov_raw[21] sh[12]
opacity_raw, a u8 label and 7 pad bytes.  Parameters are stored as f32.

``load_scene_device`` ingests a file straight into device arrays: the raw
record block is copied to HBM once and widened to the f64 structure-of-arrays
scene by one kernel (g6r_decode_records), so a multi-million-Gaussian scene
never takes the per-field numpy path.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import InvalidParameterError
from .scene import Scene

MAGIC = b"G6DS"
VERSION = 1
HEADER_BYTES = 16
META_BYTES = 19 * 8
RECORD_BYTES = 168
# field -> (float offset within the record's 40 leading f32, width)
_FIELDS = (("mu_p", 0, 3), ("mu_d", 3, 3), ("cov_raw", 6, 21), ("sh", 27, 12),
           ("opacity_raw", 39, 1))


class SceneFormatError(ValueError):
    """Bad magic, unsupported version, or truncated payload."""


def _record_view(payload: bytes, count: int):
    """(count, 40) f32 parameters and (count,) u8 labels over the record block."""
    raw = np.frombuffer(payload, dtype=np.uint8, count=count * RECORD_BYTES).reshape(count, RECORD_BYTES)
    params = raw[:, :160].view("<f4").reshape(count, 40)
    return params, raw[:, 160]


def _parse_header(blob: bytes, path):
    if len(blob) < HEADER_BYTES + META_BYTES:
        raise SceneFormatError(f"{path}: file too short for a scene header")
    magic, version, count = struct.unpack_from("<4sIQ", blob, 0)
    if magic != MAGIC:
        raise SceneFormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise SceneFormatError(f"{path}: unsupported format version {version}")
    meta = np.frombuffer(blob, dtype="<f8", count=19, offset=HEADER_BYTES)
    expected = HEADER_BYTES + META_BYTES + count * RECORD_BYTES
    if len(blob) != expected:
        raise SceneFormatError(f"{path}: payload is {len(blob)} bytes, header implies {expected}")
    return count, dict(spacing=meta[0:3].copy(), origin=meta[3:6].copy(),
                       direction=meta[6:15].reshape(3, 3).copy(),
                       spatial_scale=meta[15:18].copy(), directional_scale=float(meta[18]))


def save_scene(scene, path) -> None:
    """Write ``scene`` as G6DS (sceneio.py:52-74): parameters rounded to f32."""
    n = len(scene.mu_p)
    meta = np.concatenate([np.asarray(scene.spacing, np.float64).reshape(3),
                           np.asarray(scene.origin, np.float64).reshape(3),
                           np.asarray(scene.direction, np.float64).reshape(9),
                           np.broadcast_to(np.asarray(scene.spatial_scale, np.float64), (3,)),
                           [float(scene.directional_scale)]]).astype("<f8")
    rec = np.zeros((n, RECORD_BYTES), dtype=np.uint8)
    params = rec[:, :160].view("<f4").reshape(n, 40)
    for name, off, width in _FIELDS:
        params[:, off:off + width] = np.asarray(getattr(scene, name), np.float64).reshape(n, width)
    rec[:, 160] = np.asarray(scene.labels, np.uint8)
    with open(Path(path), "wb") as fh:
        fh.write(struct.pack("<4sIQ", MAGIC, VERSION, n))
        fh.write(meta.tobytes())
        fh.write(rec.tobytes())


def load_scene(path) -> Scene:
    """Read a G6DS file into a host Scene (sceneio.py:77-111)."""
    blob = Path(path).read_bytes()
    count, meta = _parse_header(blob, path)
    params, labels = _record_view(blob[HEADER_BYTES + META_BYTES:], count)
    arrays = {name: params[:, off:off + width].astype(np.float64).reshape((count, width) if width > 1 else (count,))
              for name, off, width in _FIELDS}
    return Scene(labels=labels.copy(), **arrays, **meta)


def load_scene_device(path, device=None):
    """Read a G6DS file into a device-resident scene (multigpu.DeviceScene):
    one host read, one H2D copy of the record block, one decode kernel."""
    import ctypes

    import torch

    from . import _native as nat
    from .multigpu import DeviceScene
    from .raster import _ptr, _require_cuda, _stream_handle

    _require_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    blob = Path(path).read_bytes()
    count, meta = _parse_header(blob, path)
    raw = torch.frombuffer(bytearray(blob[HEADER_BYTES + META_BYTES:]), dtype=torch.uint8)
    recs = raw.to(dev, non_blocking=False)
    out = [torch.empty((max(count, 1),) + s, dtype=torch.float64, device=dev)
           for s in ((3,), (3,), (21,), (12,), ())]
    labels = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        nat.check(nat.load().g6r_decode_records(count, _ptr(recs), *[_ptr(t) for t in out],
                                                _ptr(labels), _ptr(bad), _stream_handle()))
    if int(bad.item()):
        raise InvalidParameterError(f"{path}: records hold non-finite values or labels outside [1, 11]")
    mu_p, mu_d, cov_raw, sh, opacity_raw = (t[:count] for t in out)
    return DeviceScene(mu_p=mu_p, mu_d=mu_d, cov_raw=cov_raw, sh=sh, opacity_raw=opacity_raw,
                       labels=labels[:count], spatial_scale=meta["spatial_scale"],
                       directional_scale=meta["directional_scale"], spacing=meta["spacing"],
                       origin=meta["origin"], direction=meta["direction"])
