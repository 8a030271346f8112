"""ctypes binding of libg6r.so (the C ABI in include/g6r.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a) into ``paper_2505_17338_b200/_lib/libg6r.so``.  There is no fallback:
if the library is missing or fails to load, every render call raises
``NativeLibraryError``.  ctypes releases the GIL for the duration of each
foreign call, so concurrent render calls from Python threads overlap their
host-side launch work.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# G6R_LIBRARY overrides the in-tree build (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("G6R_LIBRARY") or os.path.join(HERE, "_lib", "libg6r.so")

G6R_OK = 0
G6R_EINVAL = -22
G6R_ENOSPC = -28
G6R_ECUDA = -5

REC_DOUBLES = 44
REC_COLUMNS = 22
FLAG_DEGENERATE = 0x80

CNT_DRAWN = 0
CNT_ENTRIES = 1
CNT_FATE = 2
CNT_OVERFLOW = 8
CNT_GRAD_NONFINITE = 9
NCOUNTERS = 16
NSTAGES = 4
STAGE_NAMES = ("project", "sort", "ranges", "composite")


class NativeLibraryError(RuntimeError):
    """libg6r.so is missing or could not be loaded (no CPU fallback exists)."""


class G6RError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"g6r error {code}: {message}")
        self.code = code


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
D = ctypes.c_double
SZ = ctypes.c_size_t


class Camera(ctypes.Structure):
    _fields_ = [("position", D * 3), ("rotation", D * 9), ("focal", D), ("cx", D), ("cy", D),
                ("znear", D), ("zfar", D), ("width", I32), ("height", I32)]


class Config(ctypes.Structure):
    _fields_ = [("tile_size", I32), ("precision", I32), ("low_pass", D), ("alpha_max", D),
                ("exp_mode", I32), ("reserved", I32)]


class Scene(ctypes.Structure):
    _fields_ = [("n", I64), ("records", P), ("flags", P)]


class SplatOut(ctypes.Structure):
    _fields_ = [("gids", P), ("means2d", P), ("conics", P), ("colors", P), ("alphas", P),
                ("depths", P), ("radii", P), ("stage", P)]


class Frame(ctypes.Structure):
    _fields_ = [("image", P), ("final_t", P), ("last_contrib", P), ("counters", P),
                ("entry_splat", P), ("tile_starts", P), ("rgba8", P), ("background", D * 3),
                ("host_image", P), ("host_rgba8", P)]


_SIGS = {
    "g6r_version": (ctypes.c_char_p, []),
    "g6r_last_error": (ctypes.c_char_p, []),
    "g6r_records_bytes": (SZ, [I64]),
    "g6r_workspace_bytes": (SZ, [I64, I64, I64, I32]),
    "g6r_prepare": (ctypes.c_int, [I64, P, P, P, P, P, P, P, D, I32, P, P, P, P]),
    "g6r_pack_records": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "g6r_render": (ctypes.c_int, [P, U32, P, P, P, SZ, I64, P, P, P]),
    "g6r_render_views": (ctypes.c_int, [P, U32, P, I32, P, P, SZ, I64, P, I32, P, P]),
    "g6r_profiler_create": (P, [I32]),
    "g6r_profiler_destroy": (None, [P]),
    "g6r_profiler_reset": (None, [P]),
    "g6r_profiler_read": (ctypes.c_int, [P, P, P]),
    "g6r_debug_expf": (ctypes.c_int, [I64, P, P, P]),
    "g6r_debug_exp": (ctypes.c_int, [I64, P, P, P]),
    "g6r_trace_dump": (ctypes.c_int, [ctypes.c_char_p]),
    "g6r_host_device_pointer": (ctypes.c_int, [P, P]),
    "g6r_backward_workspace_bytes": (SZ, [I64, I32, I32, I32, I64]),
    "g6r_render_backward": (ctypes.c_int, [P, U32, P, P, P, SZ, I64, P, P, P, P, P, D, I32, P, P, P,
                                           P, P, P, P, P, P]),
    "g6r_backward_forward": (ctypes.c_int, [P, U32, P, P, P, SZ, I64, P, P, P]),
    "g6r_backward_apply": (ctypes.c_int, [P, P, P, P, SZ, I64, P, P, P, P, P, D, I32, P, P, P, P,
                                          P, P, P, P]),
    "g6r_decode_records": (ctypes.c_int, [I64, P, P, P, P, P, P, P, P, P]),
    "g6r_compact_workspace_bytes": (SZ, [I64]),
    "g6r_decode_param_volume_count": (ctypes.c_int, [P, P, P, SZ, P, P]),
    "g6r_decode_param_volume": (ctypes.c_int, [P, P, I32, P, P, P, P, P, P, SZ, P, P, P, P, P, P,
                                               P]),
    "g6r_filter_rows": (ctypes.c_int, [I64, P, U32, P, P, P, P, P, P, SZ, P, P, P, P, P, P, P,
                                       P]),
    "g6r_loss_workspace_bytes": (SZ, [I32, I32]),
    "g6r_loss_grad": (ctypes.c_int, [P, P, I32, I32, I32, D, D, I32, P, P, SZ, P, P, P]),
    "g6r_adam_step": (ctypes.c_int, [I64, P, P, P, P, D, D, D, P]),
    "g6r_any_nonfinite": (ctypes.c_int, [I64, P, P, P]),
    "g6r_project": (ctypes.c_int, [P, U32, P, P, P, SZ, P, P, P]),
    "g6r_bin": (ctypes.c_int, [I64, P, P, P, I32, I32, I32, P, SZ, I64, P, P, P, P]),
    "g6r_composite": (ctypes.c_int, [I64, I32, P, P, P, P, P, P, I32, I32, I32, I32, I32, P, SZ,
                                     P, P, P, P]),
    "g6r_project_stage1": (ctypes.c_int, [I64, P, P, P, P, D, D, D, P, P, P, P, P]),
    "g6r_project_stage2": (ctypes.c_int, [I64, P, P, P, P, P, D, D, D, D, D, D, D, D, D, D, D, D,
                                          D, D, D, P, P, P, P, P, P, P]),
    "g6r_composite_backward": (ctypes.c_int, [I64, P, P, P, P, P, P, I32, I32, I32, I32, I32, P,
                                              P, P, P, P]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libg6r.so once; raise NativeLibraryError when it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != G6R_OK:
        msg = load().g6r_last_error().decode(errors="replace")
        raise G6RError(rc, msg)


def version() -> str:
    return load().g6r_version().decode()


class Profiler:
    """Per-stage CUDA-event timing of views rendered through g6r_render_views."""

    def __init__(self, max_views: int):
        self._lib = load()
        self.handle = self._lib.g6r_profiler_create(int(max_views))
        if not self.handle:
            raise G6RError(G6R_ECUDA, "g6r_profiler_create failed")

    def reset(self):
        self._lib.g6r_profiler_reset(self.handle)

    def read(self):
        ms = (ctypes.c_double * NSTAGES)()
        views = ctypes.c_int32(0)
        check(self._lib.g6r_profiler_read(self.handle, ms, ctypes.byref(views)))
        return dict(zip(STAGE_NAMES, list(ms))), int(views.value)

    def close(self):
        if self.handle:
            self._lib.g6r_profiler_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
