"""B200 drop-in for the reference renderer's Python entry points.

Same names, signatures, dataclasses and error behaviour as ``splatct.raster``
(reference raster.py:85-472): ``render``, ``render_with_state``,
``prepare_scene``, ``select_rows``, ``project_scene``, ``bin_splats``,
``composite_splats``, ``project_gaussian``, ``RenderConfig``, ``RenderStats``,
``SplatBatch``, ``TileEntries``, ``RenderState``.  Every stage runs as
hand-written sm_100a CUDA behind the C ABI in ``include/g6r.h``
(``libg6r.so``); this module only moves arrays, validates options and applies
the host-side policies the reference applies in Python.  There is no CPU
fallback: without a CUDA device or the built library every call raises.

Beyond the reference API it adds ``render_device`` (image stays in HBM, no
synchronisation) and ``render_views`` (many views of one scene in one call),
which the benchmark and the multi-GPU orbit use.

Determinism: kernels never depend on atomics for ordering (compaction and
entry offsets use an ordered scan, the sort is a stable LSD radix sort), so
results are bit-identical run to run and across concurrent callers.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .camera import Camera
from .errors import DegenerateCovarianceError, InvalidParameterError
from .scene import N_GROUPS

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise ImportError("paper_2505_17338_b200 needs torch for device memory and streams") from exc

MIN_ALPHA = 1.0 / 255.0          # raster.py:47
SH_C0 = 0.28209479177387814      # core.py:25
SH_C1 = 0.4886025119029199       # core.py:26
BACKEND = "cuda"
_BACKEND_NAMES = ("", "cuda", "cython", "python")   # reference names map onto the one CUDA path
_W_MODES = {"peak": 0, "raw": 1}


def active_backend() -> str:
    return BACKEND


@dataclass(frozen=True)
class RenderConfig:
    """Rendering knobs (raster.py:85-103).  ``threads`` is accepted and ignored;
    ``backend`` names of the reference all select the CUDA path.

    ``exp_mode`` (not in the reference) picks the f32 compositor's exp:
    ``"exact"`` restates glibc's expf, so the framebuffer is bit-identical to
    the reference's; ``"fast"`` uses the SFU ex2 (~1e-6 relative per
    contribution, every alpha-floor decision still exact), which keeps the image
    within the 1e-3 max-abs / 60 dB parity bound and leaves the sorted runs
    untouched.  f64 renders and RGBA8 frames are always exact."""

    tile_size: int = 16
    low_pass: float = 0.3
    alpha_max: float = 0.99
    w_mode: str = "peak"
    precision: str = "f32"
    threads: int = 0
    backend: str = ""
    degenerate_limit: float = 0.01
    exp_mode: str = "exact"

    def dtype(self):
        if self.precision == "f32":
            return np.float32
        if self.precision == "f64":
            return np.float64
        raise InvalidParameterError(f"precision must be 'f32' or 'f64', got {self.precision!r}")


DEFAULT_CONFIG = RenderConfig()


@dataclass
class SplatBatch:
    """Screen-space splats that survived culling, in ascending scene order."""

    gids: np.ndarray
    means2d: np.ndarray
    conics: np.ndarray
    colors: np.ndarray
    alphas: np.ndarray
    depths: np.ndarray
    radii: np.ndarray

    def __len__(self) -> int:
        return len(self.gids)


@dataclass
class Splat2D:
    mean2d: np.ndarray
    conic: np.ndarray
    color: np.ndarray
    alpha: float
    depth: float
    radii: tuple


@dataclass
class RenderStats:
    n_scene: int = 0
    n_selected: int = 0
    n_degenerate: int = 0
    n_view_degenerate: int = 0
    n_alpha_culled: int = 0
    n_depth_culled: int = 0
    n_projection_culled: int = 0
    n_viewport_culled: int = 0
    n_drawn: int = 0
    n_entries: int = 0


@dataclass
class TileEntries:
    entry_splat: np.ndarray
    tile_starts: np.ndarray
    tiles_x: int
    tiles_y: int


@dataclass
class RenderState:
    image: np.ndarray
    final_t: np.ndarray
    last_contrib: np.ndarray
    splats: SplatBatch
    entries: TileEntries
    camera: object
    config: RenderConfig
    stats: RenderStats


@dataclass
class ConditioningTerms:
    """Host view of the prepared terms (core.py:305-321), unpacked on demand."""

    adjust: np.ndarray
    precision_dd: np.ndarray
    sigma_prime: np.ndarray
    w_norm: np.ndarray
    degenerate: np.ndarray
    sigma: np.ndarray = None


# ---------------------------------------------------------------------------
# Device scene and prepared terms
# ---------------------------------------------------------------------------

def _require_cuda():
    if not torch.cuda.is_available():
        raise nat.NativeLibraryError("a CUDA device is required (no CPU fallback)")
    nat.load()


def _stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class ScenePrep:
    """Device-resident prepared scene: the 44-double records (g6r.h), the flags
    byte per Gaussian, and per-label totals/degenerate counts for the
    degenerate policy.  Created by ``prepare_scene`` and cached per scene."""

    def __init__(self, records, flags, label_counts, n, w_mode, device):
        self.records = records
        self.flags = flags
        self.label_counts = label_counts
        self.n = n
        self.w_mode = w_mode
        self.device = device
        self.entry_hint = max(1 << 20, 8 * n)
        self._host = None

    def scene_struct(self, flags=None) -> nat.Scene:
        f = self.flags if flags is None else flags
        return nat.Scene(self.n, self.records.data_ptr() if self.n else 0,
                         f.data_ptr() if self.n else 0)

    def _unpack(self):
        if self._host is None:
            n = self.n
            cols = self.records.view(nat.REC_COLUMNS, n, 2).cpu().numpy()
            r = cols.transpose(1, 0, 2).reshape(n, nat.REC_DOUBLES)
            q = r[:, 15:21]
            prec = np.empty((n, 3, 3))
            prec[:, 0, 0], prec[:, 1, 1], prec[:, 2, 2] = q[:, 0], q[:, 1], q[:, 2]
            prec[:, 0, 1] = prec[:, 1, 0] = q[:, 3]
            prec[:, 0, 2] = prec[:, 2, 0] = q[:, 4]
            prec[:, 1, 2] = prec[:, 2, 1] = q[:, 5]
            flags = self.flags.cpu().numpy()
            self._host = dict(
                terms=ConditioningTerms(adjust=r[:, 6:15].reshape(n, 3, 3).copy(),
                                        precision_dd=prec,
                                        sigma_prime=r[:, 21:30].reshape(n, 3, 3).copy(),
                                        w_norm=r[:, 43].copy(),
                                        degenerate=(flags & nat.FLAG_DEGENERATE) != 0),
                opacity=r[:, 42].copy())
        return self._host

    @property
    def terms(self) -> ConditioningTerms:
        return self._unpack()["terms"]

    @property
    def opacity(self) -> np.ndarray:
        return self._unpack()["opacity"]


class _DeviceScene:
    def __init__(self, scene, device):
        n = len(scene.mu_p)
        self.n = n

        def up(a, dt):
            if isinstance(a, torch.Tensor):   # already resident (multigpu.DeviceScene)
                return a.to(device=device, dtype=torch.from_numpy(np.zeros(0, dt)).dtype).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)

        self.mu_p = up(scene.mu_p, np.float64)
        self.mu_d = up(scene.mu_d, np.float64)
        self.cov_raw = up(scene.cov_raw, np.float64)
        self.sh = up(scene.sh, np.float64)
        self.opacity_raw = up(scene.opacity_raw, np.float64)
        self.labels = up(scene.labels, np.uint8)
        ss = np.asarray(scene.spatial_scale, dtype=np.float64)
        self.spatial_scale = np.ascontiguousarray(np.broadcast_to(ss, (3,)))
        self.directional_scale = float(scene.directional_scale)
        self.preps = {}


_CACHE = weakref.WeakKeyDictionary()
_CACHE_LOCK = threading.Lock()


def _device_scene(scene) -> _DeviceScene:
    dev = torch.cuda.current_device()
    with _CACHE_LOCK:
        per = _CACHE.get(scene)
        if per is None:
            per = {}
            _CACHE[scene] = per
        ds = per.get(dev)
        if ds is None:
            ds = _DeviceScene(scene, torch.device("cuda", dev))
            per[dev] = ds
    return ds


def prepare_scene(scene, w_mode: str = "peak") -> ScenePrep:
    """Prepared slicing terms for ``scene`` on the current device (raster.py:120-137).

    Cached on the scene object; a new Scene (e.g. after an optimizer step)
    gets a fresh upload and prep."""
    if w_mode not in _W_MODES:
        raise ValueError(f"unknown opacity modulation mode {w_mode!r}")
    _require_cuda()
    ds = _device_scene(scene)
    prep = ds.preps.get(w_mode)
    if prep is not None:
        return prep
    n = ds.n
    dev = ds.mu_p.device
    records = torch.empty(max(n, 1) * nat.REC_DOUBLES, dtype=torch.float64, device=dev)
    flags = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    counts = torch.empty(32, dtype=torch.int64, device=dev)
    ss = (ctypes.c_double * 3)(*ds.spatial_scale.tolist())
    nat.check(nat.load().g6r_prepare(
        n, _ptr(ds.mu_p), _ptr(ds.mu_d), _ptr(ds.cov_raw), _ptr(ds.sh), _ptr(ds.opacity_raw),
        _ptr(ds.labels), ctypes.cast(ss, ctypes.c_void_p), ds.directional_scale,
        _W_MODES[w_mode], _ptr(records), _ptr(flags), _ptr(counts), _stream_handle()))
    prep = ScenePrep(records, flags, counts.cpu().numpy(), n, w_mode, dev)
    ds.preps[w_mode] = prep
    return prep


def prepare_from_terms(scene, terms, opacity, device=None) -> ScenePrep:
    """Wrap externally computed terms (adjust, precision_dd, sigma_prime,
    w_norm, degenerate + opacity) as a device prep, bypassing g6r_prepare.
    Used to isolate the projection in parity checks."""
    _require_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n = len(scene.mu_p)

    def up(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)

    records = torch.empty(max(n, 1) * nat.REC_DOUBLES, dtype=torch.float64, device=dev)
    flags = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    args = [up(scene.mu_p, np.float64), up(scene.mu_d, np.float64), up(scene.sh, np.float64),
            up(opacity, np.float64), up(terms.w_norm, np.float64), up(terms.adjust, np.float64),
            up(terms.precision_dd, np.float64), up(terms.sigma_prime, np.float64),
            up(terms.degenerate, np.uint8), up(scene.labels, np.uint8)]
    nat.check(nat.load().g6r_pack_records(n, *[_ptr(a) for a in args], _ptr(records), _ptr(flags),
                                         _stream_handle()))
    labels = np.asarray(scene.labels).astype(np.int64)
    deg = np.asarray(terms.degenerate, dtype=bool)
    counts = np.zeros(32, dtype=np.int64)
    counts[:16] = np.bincount(labels, minlength=16)[:16]
    counts[16:] = np.bincount(labels[deg], minlength=16)[:16]
    return ScenePrep(records, flags, counts, n, "external", dev)


# ---------------------------------------------------------------------------
# Selection (raster.py:140-154, 418-440)
# ---------------------------------------------------------------------------

def normalize_group_mask(group_mask) -> np.ndarray:
    arr = np.asarray(group_mask)
    if arr.dtype == bool:
        if arr.shape != (N_GROUPS,):
            raise InvalidParameterError(
                f"boolean group mask must have shape ({N_GROUPS},), got {arr.shape}")
        return arr.copy()
    mask = np.zeros(N_GROUPS, dtype=bool)
    for g in np.atleast_1d(arr):
        idx = int(g)
        if not 0 <= idx < N_GROUPS:
            raise InvalidParameterError(f"group index {idx} outside [0, {N_GROUPS - 1}]")
        mask[idx] = True
    return mask


_ALL = 0xFFFF


def _selection(prep: ScenePrep, group_mask, config: RenderConfig, stats: RenderStats) -> int:
    """Mask bits for the kernels + the degenerate policy, from per-label counts
    precomputed at prep time (no per-frame device transfer)."""
    stats.n_scene = prep.n
    tot, bad = prep.label_counts[:16], prep.label_counts[16:]
    if group_mask is None:
        bits, n_sel, n_bad = _ALL, int(tot.sum()), int(bad.sum())
    else:
        m = normalize_group_mask(group_mask)
        groups = np.nonzero(m)[0]
        bits = int(sum(1 << int(g) for g in groups))
        n_sel, n_bad = int(tot[groups].sum()), int(bad[groups].sum())
    stats.n_selected = n_sel
    stats.n_degenerate = n_bad
    if n_sel and n_bad > config.degenerate_limit * n_sel:
        raise DegenerateCovarianceError(
            f"{n_bad} of {n_sel} selected Gaussians have singular directional covariance "
            f"(limit {config.degenerate_limit:.0%})")
    return bits


def select_rows(scene, prep: ScenePrep, group_mask, config: RenderConfig,
                stats: RenderStats) -> np.ndarray:
    """Group-masked, non-degenerate scene rows (host array, API parity)."""
    _selection(prep, group_mask, config, stats)
    labels = np.asarray(scene.labels)
    if group_mask is None:
        selected = np.arange(len(labels), dtype=np.int64)
    else:
        selected = np.nonzero(normalize_group_mask(group_mask)[labels])[0]
    deg = prep.terms.degenerate[selected]
    return selected[~deg]


# ---------------------------------------------------------------------------
# Camera / config structs
# ---------------------------------------------------------------------------

def _check_config(config) -> nat.Config:
    """Validate a RenderConfig -- ours, or the reference's own
    ``splatct.raster.RenderConfig`` (no ``exp_mode``: the exact path)."""
    if config.precision not in ("f32", "f64"):
        raise InvalidParameterError(f"precision must be 'f32' or 'f64', got {config.precision!r}")
    exp_mode = getattr(config, "exp_mode", "exact")
    if config.backend not in _BACKEND_NAMES:
        raise InvalidParameterError(f"unknown backend {config.backend!r}")
    if not 1 <= int(config.tile_size) <= 32:
        raise InvalidParameterError(f"tile_size must lie in [1, 32], got {config.tile_size}")
    if exp_mode not in ("exact", "fast"):
        raise InvalidParameterError(f"exp_mode must be 'exact' or 'fast', got {exp_mode!r}")
    return nat.Config(int(config.tile_size), 0 if config.precision == "f32" else 1,
                      float(config.low_pass), float(config.alpha_max),
                      1 if exp_mode == "fast" else 0, 0)


def _camera_struct(camera) -> nat.Camera:
    c = nat.Camera()
    pos = np.asarray(camera.position, dtype=np.float64)
    rot = np.asarray(camera.rotation, dtype=np.float64).reshape(9)
    c.position[:] = pos.tolist()
    c.rotation[:] = rot.tolist()
    c.focal = float(camera.focal)
    c.cx = float(camera.cx)
    c.cy = float(camera.cy)
    c.znear = float(camera.near)
    c.zfar = float(camera.far)
    c.width = int(camera.width)
    c.height = int(camera.height)
    return c


_CAMERA_DTYPE = np.dtype([("position", "<f8", (3,)), ("rotation", "<f8", (9,)), ("focal", "<f8"),
                          ("cx", "<f8"), ("cy", "<f8"), ("znear", "<f8"), ("zfar", "<f8"),
                          ("width", "<i4"), ("height", "<i4")])   # g6r_camera (g6r.h)


def _camera_array(cams):
    """The g6r_camera array of ``cams`` for one g6r_render_views call, filled
    column by column (a ctypes struct per camera costs ~1.6 us of host time
    before the GPU's first kernel)."""
    a = np.empty(len(cams), _CAMERA_DTYPE)
    a["position"] = np.array([c.position for c in cams], dtype=np.float64).reshape(-1, 3)
    a["rotation"] = np.array([c.rotation for c in cams], dtype=np.float64).reshape(-1, 9)
    a["focal"] = [c.focal for c in cams]
    a["cx"] = [c.cx for c in cams]
    a["cy"] = [c.cy for c in cams]
    a["znear"] = [c.near for c in cams]
    a["zfar"] = [c.far for c in cams]
    a["width"] = [c.width for c in cams]
    a["height"] = [c.height for c in cams]
    return a


_FRAME_DTYPE = np.dtype([("image", "<u8"), ("final_t", "<u8"), ("last_contrib", "<u8"),
                         ("counters", "<u8"), ("entry_splat", "<u8"), ("tile_starts", "<u8"),
                         ("rgba8", "<u8"), ("background", "<f8", (3,)), ("host_image", "<u8"),
                         ("host_rgba8", "<u8")])   # g6r_frame (g6r.h)


def _tiles(camera, tile_size):
    tx = (int(camera.width) + tile_size - 1) // tile_size
    ty = (int(camera.height) + tile_size - 1) // tile_size
    return tx, ty


# ---------------------------------------------------------------------------
# Frame rendering
# ---------------------------------------------------------------------------

class DeviceFrame:
    """One rendered view kept in HBM (torch tensors on the render device)."""

    def __init__(self, image, final_t, last_contrib, counters, entry_splat=None,
                 tile_starts=None, splats=None, capacity=0):
        self.image = image
        self.final_t = final_t
        self.last_contrib = last_contrib
        self.counters = counters
        self.entry_splat = entry_splat
        self.tile_starts = tile_starts
        self.splats = splats
        self.capacity = capacity


def _alloc_frame(camera, config, dev, with_state, cap, n, T, track=True):
    H, W = int(camera.height), int(camera.width)
    dt = torch.float32 if config.precision == "f32" else torch.float64
    # track=False (image only): no final_t / last_contrib, so the runs may skip
    # the entries no pixel can visit (g6r_tiles.cu part_ctx)
    fr = DeviceFrame(torch.empty((H, W, 4), dtype=dt, device=dev),
                     torch.empty((H, W), dtype=dt, device=dev) if track else None,
                     torch.empty((H, W), dtype=torch.int32, device=dev) if track else None,
                     torch.empty(nat.NCOUNTERS, dtype=torch.int64, device=dev), capacity=cap)
    if with_state:
        m = max(n, 1)
        fr.entry_splat = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        fr.tile_starts = torch.empty(T + 1, dtype=torch.int64, device=dev)
        fr.splats = dict(gids=torch.empty(m, dtype=torch.int64, device=dev),
                         means2d=torch.empty((m, 2), dtype=torch.float64, device=dev),
                         conics=torch.empty((m, 3), dtype=torch.float64, device=dev),
                         colors=torch.empty((m, 3), dtype=torch.float64, device=dev),
                         alphas=torch.empty(m, dtype=torch.float64, device=dev),
                         depths=torch.empty(m, dtype=torch.float64, device=dev),
                         radii=torch.empty((m, 2), dtype=torch.int32, device=dev))
    return fr


def _frame_struct(fr: DeviceFrame) -> nat.Frame:
    return nat.Frame(fr.image.data_ptr(),
                     fr.final_t.data_ptr() if fr.final_t is not None else 0,
                     fr.last_contrib.data_ptr() if fr.last_contrib is not None else 0,
                     fr.counters.data_ptr(),
                     fr.entry_splat.data_ptr() if fr.entry_splat is not None else 0,
                     fr.tile_starts.data_ptr() if fr.tile_starts is not None else 0)


def _splat_struct(fr: DeviceFrame):
    if fr.splats is None:
        return None
    s = fr.splats
    return nat.SplatOut(s["gids"].data_ptr(), s["means2d"].data_ptr(), s["conics"].data_ptr(),
                        s["colors"].data_ptr(), s["alphas"].data_ptr(), s["depths"].data_ptr(),
                        s["radii"].data_ptr(), 0)


def _workspace(n, T, cap, precision, dev):
    nbytes = nat.load().g6r_workspace_bytes(n, T, cap, precision)
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev), nbytes


def _launch(prep: ScenePrep, bits: int, camera, config: RenderConfig, with_state: bool,
            cap: int, track: bool = True) -> DeviceFrame:
    cfg = _check_config(config)
    cam = _camera_struct(camera)
    tx, ty = _tiles(camera, cfg.tile_size)
    T = tx * ty
    fr = _alloc_frame(camera, config, prep.device, with_state, cap, prep.n, T, track or with_state)
    ws, nbytes = _workspace(prep.n, T, cap, cfg.precision, prep.device)
    sc = prep.scene_struct()
    f = _frame_struct(fr)
    so = _splat_struct(fr)
    nat.check(nat.load().g6r_render(ctypes.byref(sc), bits, ctypes.byref(cam), ctypes.byref(cfg),
                                    _ptr(ws), nbytes, cap, ctypes.byref(f),
                                    ctypes.byref(so) if so is not None else None,
                                    _stream_handle()))
    fr._ws = ws   # keep alive until the stream has consumed it
    return fr


def _render_checked(prep, bits, camera, config, with_state):
    """Render, synchronise once, and re-render with a larger entry capacity if
    the view overflowed the current one."""
    while True:
        cap = int(prep.entry_hint)
        fr = _launch(prep, bits, camera, config, with_state, cap)
        counters = fr.counters.cpu().numpy()
        if not counters[nat.CNT_OVERFLOW]:
            return fr, counters
        prep.entry_hint = min(int(counters[nat.CNT_ENTRIES] * 1.25) + 4096, (1 << 30) - 1)


def render_device(scene, camera, group_mask=None, config: RenderConfig = DEFAULT_CONFIG,
                  capacity: int | None = None) -> DeviceFrame:
    """Enqueue one view and return its device frame without synchronising.
    ``frame.counters[8]`` (overflow) must be 0 for the frame to be valid; the
    default capacity comes from the scene's entry hint (raised by any
    synchronising render that overflowed)."""
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, RenderStats())
    return _launch(prep, bits, camera, config, False, int(capacity or prep.entry_hint))


DEFAULT_CONCURRENCY = 16  # views per batched launch (g6r_render_views)
MAX_BATCH = 16            # kMaxBatch in csrc/g6r_internal.h
PIPELINE_LANES = int(os.environ.get("G6R_LANES", "2"))   # streams batches alternate over (<= 4)
# render_batch writing the pinned host images directly from the compositor
# (G6R_ZERO_COPY=1).  Off by default: measured at cfg3 (20 views), the PCIe
# stores throttle the compositor -- 3590 views/s end to end against 3870 for
# device images + overlapped copy-engine D2H (tools/probe_e2e.py)
ZERO_COPY = os.environ.get("G6R_ZERO_COPY", "0") == "1"


def render_views(scene, cameras, group_mask=None, config: RenderConfig = DEFAULT_CONFIG,
                 capacity: int | None = None, out=None, profiler=None,
                 concurrency: int = DEFAULT_CONCURRENCY, rgba8=None, background=(0.0, 0.0, 0.0),
                 image: bool = True, pipeline: bool = True, entry_splat=None, tile_starts=None,
                 host_out=None, host_rgba8=None):
    """Render ``cameras`` (same size) with up to ``concurrency`` views in flight.

    Returns ``(images, counters)``: ``images`` (V,H,W,4) on the device,
    ``counters`` (V,16) int64.  No synchronisation; a view with
    ``counters[v, 8] != 0`` overflowed ``capacity`` and must be re-rendered.
    ``rgba8`` ((V,H,W,4) uint8 device tensor) additionally receives the served
    frame composited over ``background`` and quantised in the compositor's
    epilogue; with ``image=False`` the float image is not written at all
    (``images`` is then None).
    ``entry_splat`` ((V, capacity) int32) and ``tile_starts`` ((V, T+1) int64)
    device tensors, when given, receive every view's sorted tile runs exactly
    as ``TileEntries`` holds them (indices into the view's compacted
    SplatBatch, raster.py:201-208); entries past ``counters[v, 1]`` are
    undefined.
    ``host_out`` / ``host_rgba8`` (pinned CPU tensors shaped like the image /
    rgba8 outputs) receive each view's copy as soon as the view is complete,
    overlapped with the rest of the call (g6r_frame.host_image / host_rgba8);
    they are complete once the current stream reaches the end of the call."""
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, RenderStats())
    cfg = _check_config(config)
    cams = list(cameras)
    V = len(cams)
    H, W = int(cams[0].height), int(cams[0].width)
    if any(int(c.height) != H or int(c.width) != W for c in cams):
        raise InvalidParameterError("render_views needs cameras of one image size")
    dt = torch.float32 if config.precision == "f32" else torch.float64
    dev = prep.device
    if image:
        images = out if out is not None else torch.empty((V, H, W, 4), dtype=dt, device=dev)
    elif rgba8 is None:
        raise InvalidParameterError("image=False needs an rgba8 output")
    else:
        images = None
    if rgba8 is not None and (tuple(rgba8.shape) != (V, H, W, 4) or rgba8.dtype != torch.uint8
                              or not rgba8.is_contiguous()):
        raise InvalidParameterError(f"rgba8 must be a contiguous ({V}, {H}, {W}, 4) uint8 tensor")
    counters = torch.empty((V, nat.NCOUNTERS), dtype=torch.int64, device=dev)
    cap = int(capacity or prep.entry_hint)
    T = (lambda t: t[0] * t[1])(_tiles(cams[0], cfg.tile_size))
    if entry_splat is not None and (entry_splat.dtype != torch.int32 or not entry_splat.is_contiguous()
                                    or entry_splat.dim() != 2 or entry_splat.shape[0] != V
                                    or entry_splat.shape[1] < cap):
        raise InvalidParameterError(f"entry_splat must be a contiguous (V, >= {cap}) int32 tensor")
    if tile_starts is not None and (tile_starts.dtype != torch.int64 or not tile_starts.is_contiguous()
                                    or tuple(tile_starts.shape) != (V, T + 1)):
        raise InvalidParameterError(f"tile_starts must be a contiguous ({V}, {T + 1}) int64 tensor")
    for name, t, want in (("host_out", host_out, images), ("host_rgba8", host_rgba8, rgba8)):
        if t is None:
            continue
        if want is None or tuple(t.shape) != tuple(want.shape) or t.dtype != want.dtype \
                or not t.is_contiguous() or not t.is_pinned():
            raise InvalidParameterError(f"{name} must be a pinned contiguous CPU tensor shaped like the output")
    slots = max(1, min(int(concurrency), MAX_BATCH, V))
    if pipeline and profiler is None and 4 <= V <= slots:
        # one batch would leave nothing to overlap: two half batches pipelined
        # on two streams instead (measured 16 views at 512^2 4943 -> 4962
        # views/s, 12 at 1024^2 2751 -> 2826)
        slots = (V + 1) // 2
    tx, ty = _tiles(cams[0], cfg.tile_size)
    per = nat.load().g6r_workspace_bytes(prep.n, tx * ty, cap, cfg.precision)
    # n batches' worth of workspace pipelines consecutive batches on n streams
    lanes = PIPELINE_LANES if (V > slots and profiler is None and pipeline) else 1
    ws = torch.empty(max(per * slots * lanes, 256), dtype=torch.uint8, device=dev)
    cam_np = _camera_array(cams)
    cam_arr = (nat.Camera * V).from_buffer(cam_np)
    # per-view frames with addresses by stride arithmetic on the contiguous
    # outputs (a tensor index or a ctypes struct per view costs microseconds
    # of host time, and the host time before the first launch is GPU idle)
    if images is not None and not images.is_contiguous():
        raise InvalidParameterError("out must be a contiguous (V, H, W, 4) tensor")
    fr = np.zeros(V, _FRAME_DTYPE)
    idx = np.arange(V, dtype=np.uint64)
    for field, t in (("image", images), ("counters", counters), ("entry_splat", entry_splat),
                     ("tile_starts", tile_starts), ("rgba8", rgba8), ("host_image", host_out),
                     ("host_rgba8", host_rgba8)):
        if t is not None:
            fr[field] = np.uint64(t.data_ptr()) + idx * np.uint64(t.stride(0) * t.element_size())
    fr["background"] = [float(c) for c in background]
    frames = (nat.Frame * V).from_buffer(fr)
    sc = prep.scene_struct()
    nat.check(nat.load().g6r_render_views(ctypes.byref(sc), bits, cam_arr, V, ctypes.byref(cfg),
                                          _ptr(ws), per * slots * lanes, cap, frames, slots,
                                          profiler.handle if profiler is not None else None,
                                          _stream_handle()))
    counters._g6r_keepalive = ws
    return images, counters


def _host_mapped(t) -> bool:
    """True when pinned host tensor ``t`` is addressable by the device at its
    own address (unified addressing), so kernels can write it directly."""
    dptr = ctypes.c_void_p()
    rc = nat.load().g6r_host_device_pointer(ctypes.c_void_p(t.data_ptr()), ctypes.byref(dptr))
    return rc == 0 and dptr.value == t.data_ptr()


def render_batch(scene, cameras, group_mask=None, config: RenderConfig = DEFAULT_CONFIG,
                 batch: int = DEFAULT_CONCURRENCY) -> np.ndarray:
    """Render many views to host memory: (V, H, W, 4) like stacking
    ``render(scene, cam)`` over ``cameras``.

    One ``render_views`` call (``batch`` views per launch, consecutive batches
    pipelined on two streams) whose frames carry page-locked host
    destinations: the library copies each view device->host as soon as the
    compositor has finished it (g6r_frame.host_image, gated on the device by
    the view's completion flag), so the transfers overlap the rest of the
    rendering and only the last view's copy trails the last kernel.  One
    synchronisation at the end; views that overflowed the entry capacity are
    re-rendered individually."""
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, RenderStats())
    cams = list(cameras)
    V = len(cams)
    if V == 0:
        return np.zeros((0, 0, 0, 4), dtype=config.dtype())
    H, W = int(cams[0].height), int(cams[0].width)
    dt = torch.float32 if config.precision == "f32" else torch.float64
    # pinned output owned by the returned array (torch's caching host allocator
    # recycles the block once the array is released): no extra host copy
    host = torch.empty((V, H, W, 4), dtype=dt, pin_memory=True)
    chunk = max(1, min(int(batch), MAX_BATCH))
    if ZERO_COPY and _host_mapped(host):
        # the compositor epilogue writes the pinned host array itself
        _, cnt = render_views(scene, cams, group_mask, config, out=host, concurrency=chunk)
    else:
        _, cnt = render_views(scene, cams, group_mask, config, concurrency=chunk, host_out=host)
    cnt = cnt.cpu().numpy()   # synchronises: kernels and host copies are done
    out = host.numpy()
    for v in np.nonzero(cnt[:, nat.CNT_OVERFLOW])[0]:
        fr, _ = _render_checked(prep, bits, cams[v], config, False)
        out[v] = fr.image.cpu().numpy()
    return out


def render_frames_u8(scene, cameras, background=(0.0, 0.0, 0.0), group_mask=None,
                     config: RenderConfig = DEFAULT_CONFIG, batch: int = DEFAULT_CONCURRENCY,
                     device_out: bool = False):
    """Served frames: (V, H, W, 4) uint8 RGBA of every view composited over an
    opaque ``background`` -- exactly ``to_rgba_u8(composite_over(render(scene,
    cam), background))`` of the reference (metrics.py:21-25, _png.py:21-32) --
    produced by the compositor's epilogue, so no float image is written to HBM
    and 1 byte per channel crosses PCIe.  ``device_out`` returns the device
    tensor instead of a host array."""
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, RenderStats())
    cams = list(cameras)
    V = len(cams)
    if V == 0:
        return np.zeros((0, 0, 0, 4), dtype=np.uint8)
    H, W = int(cams[0].height), int(cams[0].width)
    dev = prep.device
    frames = torch.empty((V, H, W, 4), dtype=torch.uint8, device=dev)
    chunk = max(1, min(int(batch), MAX_BATCH))
    host = None if device_out else torch.empty((V, H, W, 4), dtype=torch.uint8, pin_memory=True)
    # each view's frame is copied to `host` as soon as it is complete
    _, cnt = render_views(scene, cams, group_mask, config, concurrency=chunk, rgba8=frames,
                          background=background, image=False, host_rgba8=host)
    cnt = cnt.cpu().numpy()   # synchronises: kernels and host copies are done
    for v in np.nonzero(cnt[:, nat.CNT_OVERFLOW])[0]:
        while True:   # re-render an overflowed view with a grown capacity
            prep.entry_hint = min(int(cnt[v, nat.CNT_ENTRIES] * 1.25) + 4096, (1 << 30) - 1)
            _, c1 = render_views(scene, [cams[v]], group_mask, config, concurrency=1,
                                 capacity=prep.entry_hint, rgba8=frames[v:v + 1],
                                 background=background, image=False)
            c1 = c1.cpu().numpy()
            if not c1[0, nat.CNT_OVERFLOW]:
                break
            cnt[v] = c1[0]
        if host is not None:
            host[v].copy_(frames[v])
    if host is None:
        return frames
    return host.numpy()


def _stats_from_counters(stats: RenderStats, counters) -> None:
    fate = counters[nat.CNT_FATE:nat.CNT_FATE + 6]
    stats.n_view_degenerate = int(fate[1])
    stats.n_alpha_culled = int(fate[2])
    stats.n_depth_culled = int(fate[3])
    stats.n_projection_culled = int(fate[4])
    stats.n_viewport_culled = int(fate[5])
    stats.n_drawn = int(counters[nat.CNT_DRAWN])
    stats.n_entries = int(counters[nat.CNT_ENTRIES])


def render_with_state(scene, camera, group_mask=None,
                      config: RenderConfig = DEFAULT_CONFIG) -> RenderState:
    """Render and return every intermediate (raster.py:443-455)."""
    stats = RenderStats()
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, stats)
    fr, counters = _render_checked(prep, bits, camera, config, True)
    _stats_from_counters(stats, counters)
    m, e = stats.n_drawn, stats.n_entries
    s = fr.splats
    splats = SplatBatch(gids=s["gids"][:m].cpu().numpy(), means2d=s["means2d"][:m].cpu().numpy(),
                        conics=s["conics"][:m].cpu().numpy(), colors=s["colors"][:m].cpu().numpy(),
                        alphas=s["alphas"][:m].cpu().numpy(), depths=s["depths"][:m].cpu().numpy(),
                        radii=s["radii"][:m].cpu().numpy())
    tx, ty = _tiles(camera, int(config.tile_size))
    entries = TileEntries(entry_splat=fr.entry_splat[:e].cpu().numpy(),
                          tile_starts=fr.tile_starts.cpu().numpy(), tiles_x=tx, tiles_y=ty)
    return RenderState(image=fr.image.cpu().numpy(), final_t=fr.final_t.cpu().numpy(),
                       last_contrib=fr.last_contrib.cpu().numpy(), splats=splats,
                       entries=entries, camera=camera, config=config, stats=stats)


def render(scene, camera, group_mask=None, config: RenderConfig = DEFAULT_CONFIG) -> np.ndarray:
    """(H, W, 4) premultiplied RGBA (raster.py:458-466)."""
    prep = prepare_scene(scene, config.w_mode)
    bits = _selection(prep, group_mask, config, RenderStats())
    while True:
        fr = _launch(prep, bits, camera, config, False, int(prep.entry_hint), track=False)
        # image and counters come back in one synchronisation, via pinned memory
        img = torch.empty(fr.image.shape, dtype=fr.image.dtype, pin_memory=True)
        cnt = torch.empty(nat.NCOUNTERS, dtype=torch.int64, pin_memory=True)
        img.copy_(fr.image, non_blocking=True)
        cnt.copy_(fr.counters, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        c = cnt.numpy()
        if not c[nat.CNT_OVERFLOW]:
            return img.numpy()
        prep.entry_hint = min(int(c[nat.CNT_ENTRIES] * 1.25) + 4096, (1 << 30) - 1)


# ---------------------------------------------------------------------------
# Stage helpers (bench.py:26-36 uses them): device work, host arrays in/out
# ---------------------------------------------------------------------------

def project_scene(scene, prep: ScenePrep, rows, camera, config: RenderConfig,
                  stats: RenderStats) -> SplatBatch:
    """Project scene rows ``rows`` (degenerate-free, ascending) into splats."""
    cfg = _check_config(config)
    cam = _camera_struct(camera)
    rows = np.asarray(rows, dtype=np.int64)
    n = prep.n
    dev = prep.device
    flags = prep.flags
    bits = _ALL
    if rows.size != n:
        sel = np.zeros(n, dtype=bool)
        sel[rows] = True
        off = torch.from_numpy(~sel).to(dev)
        flags = torch.where(off, (prep.flags & nat.FLAG_DEGENERATE) | 15, prep.flags)
        bits = _ALL & ~(1 << 15)
    fr = _alloc_frame(camera, config, dev, True, 1, n, 1)
    counters = fr.counters
    stage = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    so = _splat_struct(fr)
    so.stage = stage.data_ptr()
    tx, ty = _tiles(camera, cfg.tile_size)
    ws, nbytes = _workspace(n, tx * ty, 0, cfg.precision, dev)
    sc = prep.scene_struct(flags)
    nat.check(nat.load().g6r_project(ctypes.byref(sc), bits, ctypes.byref(cam), ctypes.byref(cfg),
                                     _ptr(ws), nbytes, _ptr(counters), ctypes.byref(so),
                                     _stream_handle()))
    c = counters.cpu().numpy()
    _stats_from_counters(stats, c)
    stats.n_entries = 0
    m = int(c[nat.CNT_DRAWN])
    s = fr.splats
    return SplatBatch(gids=s["gids"][:m].cpu().numpy(), means2d=s["means2d"][:m].cpu().numpy(),
                      conics=s["conics"][:m].cpu().numpy(), colors=s["colors"][:m].cpu().numpy(),
                      alphas=s["alphas"][:m].cpu().numpy(), depths=s["depths"][:m].cpu().numpy(),
                      radii=s["radii"][:m].cpu().numpy())


def project_gaussian(gaussian, camera, spatial_scale=1.0, directional_scale=1.0,
                     config: RenderConfig = DEFAULT_CONFIG):
    """Project one 6D Gaussian; None when culled (raster.py:312-337)."""
    from .scene import Scene
    sc = Scene(mu_p=np.asarray(gaussian.mu_p, dtype=np.float64)[None, :],
               mu_d=np.asarray(gaussian.mu_d, dtype=np.float64)[None, :],
               cov_raw=np.asarray(gaussian.cov_raw, dtype=np.float64)[None, :],
               sh=np.asarray(gaussian.sh, dtype=np.float64)[None, :],
               opacity_raw=np.asarray([gaussian.opacity_raw], dtype=np.float64),
               labels=np.array([max(1, int(getattr(gaussian, "label", 1) or 1))]),
               spatial_scale=np.broadcast_to(np.asarray(spatial_scale, dtype=np.float64), (3,)),
               directional_scale=directional_scale)
    prep = prepare_scene(sc, config.w_mode)
    if prep.label_counts[16:].sum():
        raise DegenerateCovarianceError("directional covariance block is singular")
    stats = RenderStats(n_scene=1, n_selected=1)
    sp = project_scene(sc, prep, np.arange(1), camera, config, stats)
    if len(sp) == 0:
        return None
    return Splat2D(mean2d=sp.means2d[0], conic=sp.conics[0], color=sp.colors[0],
                   alpha=float(sp.alphas[0]), depth=float(sp.depths[0]),
                   radii=(int(sp.radii[0, 0]), int(sp.radii[0, 1])))


def bin_splats(splats: SplatBatch, camera, tile_size: int) -> TileEntries:
    """Duplicate splats into overlapped tiles and depth-sort (raster.py:340-381)."""
    _require_cuda()
    if not 1 <= int(tile_size):
        raise InvalidParameterError(f"tile_size must be positive, got {tile_size}")
    dev = torch.device("cuda", torch.cuda.current_device())
    tx, ty = _tiles(camera, int(tile_size))
    T = tx * ty
    m = len(splats.depths)
    means2d = torch.from_numpy(np.ascontiguousarray(splats.means2d, np.float64).reshape(-1, 2)).to(dev)
    radii = torch.from_numpy(np.ascontiguousarray(splats.radii, np.int32).reshape(-1, 2)).to(dev)
    depths = torch.from_numpy(np.ascontiguousarray(splats.depths, np.float64)).to(dev)
    counters = torch.empty(nat.NCOUNTERS, dtype=torch.int64, device=dev)
    starts = torch.empty(T + 1, dtype=torch.int64, device=dev)
    cap = max(1 << 16, 8 * m)
    while True:
        es = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        ws, nbytes = _workspace(m, T, cap, 0, dev)
        nat.check(nat.load().g6r_bin(m, _ptr(means2d), _ptr(radii), _ptr(depths),
                                     int(camera.width), int(camera.height), int(tile_size),
                                     _ptr(ws), nbytes, cap, _ptr(es), _ptr(starts), _ptr(counters),
                                     _stream_handle()))
        c = counters.cpu().numpy()
        if not c[nat.CNT_OVERFLOW]:
            break
        cap = int(c[nat.CNT_ENTRIES]) + 1
    e = int(c[nat.CNT_ENTRIES])
    return TileEntries(entry_splat=es[:e].cpu().numpy(), tile_starts=starts.cpu().numpy(),
                       tiles_x=tx, tiles_y=ty)


def composite_splats(splats: SplatBatch, entries: TileEntries, camera,
                     config: RenderConfig = DEFAULT_CONFIG):
    """Composite pre-binned splats (raster.py:469-472) -> (image, final_t, last_contrib)."""
    cfg = _check_config(config)
    dt = np.float32 if config.precision == "f32" else np.float64
    return composite_arrays(splats.means2d, splats.conics, splats.colors, splats.alphas,
                            entries.entry_splat, entries.tile_starts, entries.tiles_x,
                            cfg.tile_size, int(camera.height), int(camera.width), dt)


def composite_arrays(means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
                     tile_size, height, width, dtype):
    """Composite reference-shaped host arrays on the device (the kernel-module
    contract of _kernels.pyx:36-105); returns host (image, final_t, last)."""
    _require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    prec = 0 if np.dtype(dtype) == np.float32 else 1
    tdt = torch.float32 if prec == 0 else torch.float64

    def up(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)

    m = len(np.asarray(alphas))
    args = [up(np.asarray(means2d).reshape(-1, 2), dtype), up(np.asarray(conics).reshape(-1, 3), dtype),
            up(np.asarray(colors).reshape(-1, 3), dtype), up(alphas, dtype)]
    es = up(entry_splat, np.int32)
    ts = up(tile_starts, np.int64)
    tiles_y = (height + tile_size - 1) // tile_size
    if tiles_x != (width + tile_size - 1) // tile_size or len(tile_starts) != tiles_x * tiles_y + 1:
        raise InvalidParameterError("tile_starts/tiles_x do not match the framebuffer size")
    image = torch.zeros((height, width, 4), dtype=tdt, device=dev)
    final_t = torch.ones((height, width), dtype=tdt, device=dev)
    last = torch.zeros((height, width), dtype=torch.int32, device=dev)
    ws, nbytes = _workspace(m, tiles_x * tiles_y, 0, prec, dev)
    nat.check(nat.load().g6r_composite(m, prec, *[_ptr(a) for a in args], _ptr(es), _ptr(ts),
                                       tiles_x, tiles_y, tile_size, width, height, _ptr(ws), nbytes,
                                       _ptr(image), _ptr(final_t), _ptr(last), _stream_handle()))
    return image.cpu().numpy(), final_t.cpu().numpy(), last.cpu().numpy()
