"""Put the B200 render path under the UNMODIFIED reference package.

The reference's callers bind ``render`` and friends by name at import time
(``service.py:34``, ``cli.py:32``, ``metrics.py:16``, ``bench.py:26-36``,
``diffrender.py:43-50``), so rebinding ``splatct.raster.render`` alone does not
reach them.  ``install()`` rebinds every such name in every splatct module that
holds one, adds a ``"cuda"`` branch to ``_kernels_for`` (``raster.py:73-82``),
and makes the errors the B200 path raises instances of the reference's own
classes (``core.py:42-51``), so ``cli.main`` maps them to the same exit codes
(``cli.py:306-319``) and callers' ``except`` clauses keep working::

    import splatct
    from paper_2505_17338_b200 import integrate
    shim = integrate.install()          # or: with integrate.install(): ...
    splatct.service.render_request_png(scene, request)   # rendered on the GPU
    shim.uninstall()

``install(kernel_modules=True)`` additionally points the reference's kernel
modules (``splatct._kernels`` / ``splatct._kernels_py``) at the kernel-module
adapter (``kernels.py``), which is how the reference's own kernel-level tests
are run against the CUDA path (tests/test_gpu_integrate.py).

Nothing here is a fallback: every rebound call runs the CUDA path and raises
``NativeLibraryError`` when the library or the GPU is missing.
"""

from __future__ import annotations

import functools
import importlib
import sys

from . import diffrender, errors, kernels, raster

# reference module -> names it binds at import time that the B200 path replaces
_REBIND = {
    "splatct.raster": ("render", "render_with_state", "prepare_scene", "select_rows",
                       "project_scene", "project_gaussian", "bin_splats", "composite_splats"),
    "splatct.service": ("render",),
    "splatct.metrics": ("render",),
    "splatct.cli": ("render", "finetune"),
    "splatct.bench": ("render", "prepare_scene", "select_rows", "project_scene", "bin_splats",
                      "composite_splats"),
    "splatct.diffrender": ("render_with_state", "prepare_scene", "render_backward", "finetune"),
}

_OURS = {
    "render": raster.render,
    "render_with_state": raster.render_with_state,
    "prepare_scene": raster.prepare_scene,
    "select_rows": raster.select_rows,
    "project_scene": raster.project_scene,
    "project_gaussian": raster.project_gaussian,
    "bin_splats": raster.bin_splats,
    "composite_splats": raster.composite_splats,
    "render_backward": diffrender.render_backward,
    "finetune": diffrender.finetune,
}

# (ours, the reference class name in splatct.core)
_ERRORS = ((errors.InvalidParameterError, "InvalidParameterError"),
           (errors.DegenerateCovarianceError, "DegenerateCovarianceError"),
           (errors.DegenerateGeometryError, "DegenerateGeometryError"))


def _dual_classes(core):
    """Subclasses of both the reference's and our exception class: caught by
    ``except splatct.core.X`` and by ``except paper_2505_17338_b200.errors.X``."""
    out = {}
    for ours, name in _ERRORS:
        theirs = getattr(core, name)
        out[ours] = type(name, (theirs, ours), {"__module__": theirs.__module__,
                                                "__doc__": theirs.__doc__})
    return out


def _translating(fn, duals):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except tuple(duals) as exc:
            for ours, dual in duals.items():
                if isinstance(exc, ours) and not isinstance(exc, dual):
                    raise dual(*exc.args).with_traceback(exc.__traceback__) from None
            raise
    call.__wrapped_b200__ = fn
    return call


class Installation:
    """Handle returned by ``install``: ``uninstall()`` restores every name
    (also usable as a context manager)."""

    def __init__(self):
        self._saved = []   # (module, name, had_attr, old value)
        self._modules = {}
        self.active = False

    def _set(self, mod, name, value):
        self._saved.append((mod, name, hasattr(mod, name), getattr(mod, name, None)))
        setattr(mod, name, value)

    def _set_module(self, key, value):
        self._modules.setdefault(key, sys.modules.get(key))
        sys.modules[key] = value

    def uninstall(self):
        for mod, name, had, old in reversed(self._saved):
            if had:
                setattr(mod, name, old)
            else:
                delattr(mod, name)
        for key, old in self._modules.items():
            if old is None:
                sys.modules.pop(key, None)
            else:
                sys.modules[key] = old
        self._saved.clear()
        self._modules.clear()
        self.active = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()
        return False


def install(package: str = "splatct", kernel_modules: bool = False) -> Installation:
    """Rebind the reference package's render entry points to the B200 path.

    ``package`` is the import name of the reference (``splatct``); its
    submodules are imported here so that every name bound at import time is
    rebound.  ``kernel_modules=True`` also replaces the reference's kernel
    modules by the CUDA kernel-module adapter (for the reference's own
    kernel-level tests)."""
    core = importlib.import_module(f"{package}.core")
    duals = _dual_classes(core)
    inst = Installation()
    wrapped = {name: _translating(fn, duals) for name, fn in _OURS.items()}
    for modname, names in _REBIND.items():
        modname = package + modname[len("splatct"):]
        try:
            mod = importlib.import_module(modname)
        except ImportError:   # a caller module the installed reference lacks
            continue
        for name in names:
            if hasattr(mod, name):
                inst._set(mod, name, wrapped[name])
    ref_raster = importlib.import_module(f"{package}.raster")
    ref_diff = importlib.import_module(f"{package}.diffrender")
    original = ref_raster._kernels_for

    def kernels_for(backend):
        if backend == "cuda" or kernel_modules:
            return kernels
        return original(backend)

    for mod in (ref_raster, ref_diff):
        if hasattr(mod, "_kernels_for"):
            inst._set(mod, "_kernels_for", kernels_for)
    if kernel_modules:
        pkg = importlib.import_module(package)
        for sub in ("_kernels", "_kernels_py"):
            inst._set_module(f"{package}.{sub}", kernels)
            inst._set(pkg, sub, kernels)
        inst._set(ref_raster, "_DEFAULT_KERNELS", kernels)
    inst.active = True
    return inst
