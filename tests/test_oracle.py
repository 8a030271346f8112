"""The CPU oracle is pinned before it is trusted (CPU-only tests).

1. Against the golden fixtures made by the unmodified reference
   (tests/golden/make_golden.py): every stage output bit for bit.
2. Against the compiled reference itself (oracle/_ref), when it was built
   here: random scenes, masks, raw mode, config-1 size.
3. The glibc expf model the f32 compositor uses, against the host libm.
"""

import ctypes
import glob
import os

import numpy as np
import pytest

from paper_2505_17338_b200 import scenes
from paper_2505_17338_b200.camera import Camera
from paper_2505_17338_b200.scene import Scene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
               if os.path.basename(p)[:-4] not in ("expf_glibc", "loss")
               and not os.path.basename(p).startswith(("bwd_", "ft_", "ingest_")))


def load_case(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    scene = Scene(mu_p=z["mu_p"], mu_d=z["mu_d"], cov_raw=z["cov_raw"], sh=z["sh"],
                  opacity_raw=z["opacity_raw"], labels=z["labels"],
                  spatial_scale=z["spatial_scale"], directional_scale=float(z["directional_scale"]))
    w, h = (int(v) for v in z["cam_wh"])
    cam = Camera(position=z["cam_position"], rotation=z["cam_rotation"], fov_y=float(z["cam_fov"]),
                 width=w, height=h)
    tile, raw = (int(v) for v in z["config"])
    return z, scene, cam, tile, "raw" if raw else "peak"


def test_golden_cases_present():
    assert len(CASES) >= 7


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_golden(oracle, name):
    z, scene, cam, tile, w_mode = load_case(name)
    prep = oracle.prepare(scene, w_mode)
    for f in ("adjust", "precision_dd", "sigma_prime", "w_norm", "degenerate"):
        np.testing.assert_array_equal(getattr(prep, f), z[f"prep_{f}"], err_msg=f)
    np.testing.assert_array_equal(prep.opacity, z["prep_opacity"])
    for prec in ("f32", "f64"):
        st = oracle.render_with_state(scene, cam, None, prec, w_mode=w_mode, tile_size=tile)
        np.testing.assert_array_equal(st.image, z[f"{prec}_image"])
        np.testing.assert_array_equal(st.final_t, z[f"{prec}_final_t"])
        np.testing.assert_array_equal(st.last_contrib, z[f"{prec}_last_contrib"])
    for f in ("gids", "means2d", "conics", "colors", "alphas", "depths", "radii"):
        np.testing.assert_array_equal(getattr(st.splats, f), z[f"splat_{f}"], err_msg=f)
    np.testing.assert_array_equal(st.entries.entry_splat, z["entry_splat"])
    np.testing.assert_array_equal(st.entries.tile_starts, z["tile_starts"])
    stats = z["stats"]
    assert len(st.splats.gids) == stats[0]
    assert len(st.entries.entry_splat) == stats[1]
    np.testing.assert_array_equal(st.fate[1:6], stats[2:7])


def test_expf_model_matches_golden_libm(oracle):
    z = np.load(os.path.join(GOLDEN, "expf_glibc.npz"))
    np.testing.assert_array_equal(oracle.expf_glibc(z["x"]), z["y"])


def test_expf_model_matches_host_libm_dense(oracle):
    # every float in [-4.5, -4.0] and [-1e-3, 0] plus a random sample of the range
    libm = ctypes.CDLL("libm.so.6")
    libm.expf.restype = ctypes.c_float
    libm.expf.argtypes = [ctypes.c_float]
    rng = np.random.default_rng(5)
    x = rng.uniform(-4.5, 0.0, 30000).astype(np.float32)
    y = np.array([libm.expf(float(v)) for v in x], dtype=np.float32)
    np.testing.assert_array_equal(oracle.expf_glibc(x), y)


def test_oracle_matches_reference_live(oracle, ref):
    from splatct import raster as R
    from splatct.priming import Scene as RS
    for seed, n, size, w_mode, mask in [(0, 300, (64, 48), "peak", None),
                                         (1, 2000, (96, 96), "raw", None),
                                         (2, 1500, (80, 64), "peak", [2, 5, 7]),
                                         (3, 10_000, (128, 128), "peak", None)]:
        s = scenes.random_scene(np.random.default_rng(seed), n)
        rs = RS(mu_p=s.mu_p, mu_d=s.mu_d, cov_raw=s.cov_raw, sh=s.sh, opacity_raw=s.opacity_raw,
                labels=s.labels, spacing=s.spacing, origin=s.origin, direction=s.direction,
                spatial_scale=s.spatial_scale)
        cam = scenes.orbit_camera(azimuth=0.4 * seed, elevation=0.1, width=size[0], height=size[1])
        for prec in ("f32", "f64"):
            want = R.render_with_state(rs, cam, mask, R.RenderConfig(precision=prec, w_mode=w_mode))
            got = oracle.render_with_state(s, cam, mask, prec, w_mode=w_mode)
            np.testing.assert_array_equal(got.image, want.image)
            np.testing.assert_array_equal(got.last_contrib, want.last_contrib)
            np.testing.assert_array_equal(got.entries.entry_splat, want.entries.entry_splat)
            np.testing.assert_array_equal(got.entries.tile_starts, want.entries.tile_starts)


def test_oracle_backward_matches_reference_kernel(oracle, ref):
    from splatct import _kernels_py as K
    z, scene, cam, tile, w_mode = load_case("rand40")
    st = oracle.render_with_state(scene, cam, None, "f64")
    s, en = st.splats, st.entries
    g = np.random.default_rng(1).normal(size=st.image.shape)
    want = np.zeros((len(en.entry_splat), 9))
    K.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat, en.tile_starts,
                         en.tiles_x, 16, st.final_t, st.last_contrib, g, want)
    got = oracle.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat,
                                    en.tile_starts, en.tiles_x, 16, cam.width, cam.height,
                                    st.final_t, st.last_contrib, g)
    np.testing.assert_array_equal(got, want)


def test_loss_oracle_matches_golden(oracle):
    """oracle.loss_parts against the reference's _loss_parts (tests/golden/loss.npz)."""
    from cases import LOSS_CASES, loss_images, oracle_kwargs
    z = np.load(os.path.join(GOLDEN, "loss.npz"))
    for i, (name, h, w, tc, kw) in enumerate(LOSS_CASES):
        p, g = loss_images(700 + i, h, w, tc)
        total, l1, ssim_loss, grad = oracle.loss_parts(p, g, **oracle_kwargs(kw))
        np.testing.assert_allclose([total, l1, ssim_loss], z[f"{name}_parts"], rtol=1e-13, atol=1e-15)
        gs = grad.reshape(-1)[z[f"{name}_idx"]]
        np.testing.assert_allclose(gs, z[f"{name}_grad_sample"], rtol=1e-9,
                                   atol=1e-12 * np.abs(gs).max())
        np.testing.assert_allclose(np.abs(grad).sum(axis=(0, 1)), z[f"{name}_grad_abs"], rtol=1e-10)


@pytest.mark.parametrize("case", ["identity", "rotated"])
def test_decode_oracle_matches_golden(oracle, case):
    from cases import INGEST_CASES, ingest_inputs
    (name, dims, seed, rotated), = [c for c in INGEST_CASES if c[0] == case]
    psi, in6, labels, spacing, origin, direction = ingest_inputs(dims, seed, rotated)
    got = oracle.decode_param_volume(psi, in6, labels, spacing, origin, direction)
    z = np.load(os.path.join(GOLDEN, f"ingest_{name}.npz"))
    for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
        np.testing.assert_array_equal(got[k], z[k], err_msg=k)
