"""Host logic of the drop-in shim (no GPU needed): which names install()
rebinds in the unmodified reference package, that uninstall() restores them
exactly, that errors are translated into the reference's classes, and that
the kernel-module replacement is undone."""

import sys

import pytest

from paper_2505_17338_b200 import errors, integrate, kernels, raster


MODULES = ("raster", "service", "metrics", "cli", "bench", "diffrender")


def snapshot(ref):
    import importlib
    out = {}
    for m in MODULES:
        mod = importlib.import_module(f"splatct.{m}")
        for name in integrate._REBIND[f"splatct.{m}"] + ("_kernels_for",):
            if hasattr(mod, name):
                out[(m, name)] = getattr(mod, name)
    return out


def test_install_rebinds_import_bound_names_and_restores(ref):
    before = snapshot(ref)
    assert before[("service", "render")] is ref.raster.render   # bound at import
    with integrate.install() as shim:
        assert shim.active
        for (m, name), old in before.items():
            new = getattr(sys.modules[f"splatct.{m}"], name)
            assert new is not old, (m, name)
            if name != "_kernels_for":
                assert new.__wrapped_b200__ is integrate._OURS[name]
        assert sys.modules["splatct.service"].render.__wrapped_b200__ is raster.render
        assert ref.raster._kernels_for("cuda") is kernels
        assert ref.raster._kernels_for("python").BACKEND == "python"
    after = snapshot(ref)
    assert after == before


def test_kernel_modules_replaced_and_restored(ref):
    orig_py = sys.modules["splatct._kernels_py"] if "splatct._kernels_py" in sys.modules else None
    with integrate.install(kernel_modules=True):
        assert sys.modules["splatct._kernels_py"] is kernels
        from splatct import _kernels_py
        assert _kernels_py is kernels
        assert ref.raster._kernels_for("python") is kernels
        assert ref.raster.active_backend() == "cuda"
    assert sys.modules.get("splatct._kernels_py") is orig_py
    assert ref.raster.active_backend() in ("cython", "python")


def test_errors_translated_to_reference_classes(ref):
    duals = integrate._dual_classes(ref.core)

    def boom(kind):
        raise kind("bad thing")

    wrapped = integrate._translating(boom, duals)
    for ours, name in integrate._ERRORS:
        with pytest.raises(getattr(ref.core, name)) as ei:
            wrapped(ours)
        assert isinstance(ei.value, ours)
        assert str(ei.value) == "bad thing"
    with pytest.raises(KeyError):   # anything else passes through untouched
        wrapped(KeyError)
    # the CLI's exit-code mapping keys on these bases
    assert issubclass(duals[errors.DegenerateCovarianceError], ArithmeticError)
    assert issubclass(duals[errors.InvalidParameterError], ValueError)


def test_reference_render_config_is_accepted(ref):
    """The reference's own RenderConfig has no exp_mode: it selects the exact
    (bit-identical) compositor."""
    cfg = raster._check_config(ref.raster.DEFAULT_CONFIG)
    assert (cfg.tile_size, cfg.precision, cfg.exp_mode) == (16, 0, 0)
    cfg = raster._check_config(ref.raster.RenderConfig(precision="f64", tile_size=8))
    assert (cfg.tile_size, cfg.precision) == (8, 1)
    with pytest.raises(errors.InvalidParameterError):
        raster._check_config(ref.raster.RenderConfig(precision="f16"))
