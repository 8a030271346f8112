"""Unchanged reference callers on the B200 path (SURVEY.md 8b "Callers").

``paper_2505_17338_b200.integrate.install()`` rebinds the render entry points
inside the UNMODIFIED reference package (oracle/_ref); these tests then drive
the reference's own callers and compare with the same calls on the reference's
CPU path:

* ``service.render_request_png`` (service.py:175-184): byte-identical PNGs;
* ``metrics.evaluate`` (metrics.py:98-120): identical report rows;
* ``cli.main`` (cli.py:160-169, 300-319): same exit codes, same PNG bytes;
* errors are ``splatct.core`` classes (core.py:42-51);
* the reference's OWN test files (tests/test_raster.py, test_acceptance.py,
  copied unmodified into oracle/_ref/ref_tests by oracle/build_ref.sh) pass
  with every render and kernel-module call routed to the CUDA path.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REF_DIR, ROOT

pytestmark = pytest.mark.gpu
REF_TESTS = os.path.join(REF_DIR, "ref_tests")


@pytest.fixture(scope="module")
def splat(ref):
    import splatct.cli  # noqa: F401
    import splatct.metrics  # noqa: F401
    import splatct.service  # noqa: F401
    return ref


def ref_scene(ref, seed, n):
    from paper_2505_17338_b200 import scenes
    s = scenes.random_scene(np.random.default_rng(seed), n)
    return ref.priming.Scene(mu_p=s.mu_p, mu_d=s.mu_d, cov_raw=s.cov_raw, sh=s.sh,
                             opacity_raw=s.opacity_raw, labels=s.labels, spacing=np.ones(3),
                             origin=np.zeros(3), direction=np.eye(3),
                             spatial_scale=np.full(3, 3.0))


def requests(ref):
    R = ref.service.RenderRequest
    return [R(position=(0.0, 12.0, -70.0), target=(0.0, 0.0, 0.0), width=128, height=96),
            R(position=(55.0, -20.0, 40.0), target=(1.0, 2.0, 0.5), fov_y=0.6, width=160,
              height=160, group_mask=0b000010100100, background=(0.2, 0.4, 0.9)),
            R(position=(-30.0, 60.0, 25.0), target=(0.0, 0.0, 0.0), width=77, height=51,
              group_mask=0)]


def test_service_png_bytes_identical(splat):
    from paper_2505_17338_b200 import integrate
    scene = ref_scene(splat, 1, 3000)
    cfgs = [splat.raster.RenderConfig(), splat.raster.RenderConfig(precision="f64")]
    want = [splat.service.render_request_png(scene, r, c) for r in requests(splat) for c in cfgs]
    with integrate.install():
        got = [splat.service.render_request_png(scene, r, c) for r in requests(splat) for c in cfgs]
        assert splat.service.render.__wrapped_b200__.__module__ == "paper_2505_17338_b200.raster"
    assert got == want
    assert splat.service.render.__module__ == "splatct.raster"   # restored


def test_metrics_evaluate_rows_identical(splat):
    from paper_2505_17338_b200 import integrate
    scene = ref_scene(splat, 2, 2500)
    cams = [r.camera() for r in requests(splat)[:2]]
    rng = np.random.default_rng(0)
    views = [(c, rng.uniform(0, 1, (c.height, c.width, 3))) for c in cams]
    want = splat.metrics.evaluate(scene, views, quantize=True).rows()
    with integrate.install():
        got = splat.metrics.evaluate(scene, views, quantize=True).rows()
    assert got == want


def test_cli_render_exit_codes_and_bytes(splat, tmp_path):
    from paper_2505_17338_b200 import integrate
    good = ref_scene(splat, 3, 2000)
    cov = good.cov_raw.copy()
    cov[:100, 3:6] = -300.0   # singular directional blocks: > 1 % degenerate
    cov[:100, 9:] = 0.0
    bad = good.with_params(cov_raw=cov)
    splat.sceneio.save_scene(good, tmp_path / "good.g6ds")
    splat.sceneio.save_scene(bad, tmp_path / "bad.g6ds")
    args = ["--position", "0,10,-70", "--target", "0,0,0", "--width", "96", "--height", "80",
            "--background", "0.1,0.2,0.3"]

    def run(tag):
        rcs = [splat.cli.main(["render", str(tmp_path / "good.g6ds"), str(tmp_path / f"{tag}.png"),
                               *args]),
               splat.cli.main(["render", str(tmp_path / "bad.g6ds"), str(tmp_path / "x.png"),
                               *args]),
               splat.cli.main(["render", str(tmp_path / "missing.g6ds"), str(tmp_path / "y.png"),
                               *args])]
        return rcs, (tmp_path / f"{tag}.png").read_bytes()

    want_rc, want_png = run("cpu")
    with integrate.install():
        got_rc, got_png = run("gpu")
    assert want_rc == [0, splat.cli.EXIT_NUMERICAL, splat.cli.EXIT_IO]
    assert got_rc == want_rc
    assert got_png == want_png


def test_errors_are_reference_classes(splat):
    from paper_2505_17338_b200 import errors, integrate
    scene = ref_scene(splat, 4, 500)
    cam = requests(splat)[0].camera()
    with integrate.install():
        with pytest.raises(splat.core.InvalidParameterError) as ei:
            splat.raster.render(scene, cam, group_mask=[99])
        assert isinstance(ei.value, errors.InvalidParameterError)
        with pytest.raises(splat.core.InvalidParameterError):
            splat.raster.render(scene, cam, config=splat.raster.RenderConfig(precision="f16"))
        cov = scene.cov_raw.copy()
        cov[:50, 3:6] = -300.0
        cov[:50, 9:] = 0.0
        with pytest.raises(splat.core.DegenerateCovarianceError):
            splat.raster.render(scene.with_params(cov_raw=cov), cam)
        # the reference's kernel selector grew a "cuda" branch
        from paper_2505_17338_b200 import kernels
        assert splat.raster._kernels_for("cuda") is kernels


def test_finetune_through_reference_cli_module(splat):
    """diffrender.finetune as the CLI binds it runs the device loop and keeps
    the reference's Scene type."""
    from paper_2505_17338_b200 import integrate
    scene = ref_scene(splat, 5, 400)
    cams = [r.camera() for r in requests(splat)[:2]]
    views = [(c, np.full((c.height, c.width, 3), 0.3)) for c in cams]
    want_scene, want_hist = splat.diffrender.finetune(scene, views, iters=3, seed=1)
    with integrate.install():
        got_scene, got_hist = splat.cli.finetune(scene, views, iters=3, seed=1)
    assert type(got_scene) is type(scene)
    assert [h["iteration"] for h in got_hist] == [h["iteration"] for h in want_hist]
    for a, b in zip(got_hist, want_hist):
        assert a["lr"] == b["lr"]
        assert a["total"] == pytest.approx(b["total"], rel=1e-8)
    np.testing.assert_allclose(got_scene.mu_p, want_scene.mu_p, rtol=1e-6, atol=1e-12)


REF_SUITES = ["test_raster.py", "test_acceptance.py", "test_service.py", "test_metrics.py",
              "test_diffrender.py"]


@pytest.mark.parametrize("suite", REF_SUITES)
def test_reference_own_suite_on_cuda(suite):
    """The reference's own test file, unmodified, with integrate.install(
    kernel_modules=True) active from pytest_configure: every render and every
    kernel-module call (both 'python' and 'cython' backends) runs on the GPU."""
    path = os.path.join(REF_TESTS, suite)
    if not os.path.isfile(path):
        pytest.skip("reference tests not copied into oracle/_ref/ref_tests")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), REF_DIR, REF_TESTS,
                                         env.get("PYTHONPATH", "")])
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "g6r_ref_plugin",
                          "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-o", "addopts=",
                          path], env=env, cwd=REF_TESTS, capture_output=True, text=True,
                         timeout=1500)
    tail = (out.stdout + out.stderr)[-4000:]
    assert out.returncode == 0, tail
    assert "[g6r] reference suite routed to the CUDA path" in out.stdout + out.stderr, tail
