"""Seeded sweep over the render path's knobs against the CPU oracle: scene size
and spread, isotropic/anisotropic covariances, opacity range, image shape, tile
size, camera pose, group mask, precision and exp mode.  Every case compares the
sorted runs and the f32 framebuffer bit for bit (exact exp), the f64 image and
the fast-exp image within the parity bound, and the drawn/entry counts, through
render_with_state (entry sort) and render_views (splat-level sort)."""
import math

import numpy as np
import pytest

from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig
from paper_2505_17338_b200.scene import filter_scene

from test_gpu_parity import assert_image_close

pytestmark = pytest.mark.gpu

CASES = list(range(64))


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 7, 300, 2500, 12000]))
    box = float(rng.uniform(2.0, 30.0))
    s = scenes.random_scene(rng, n, box=box, iso=bool(rng.integers(2)),
                            opacity_lo=float(rng.uniform(-3.0, 0.5)), opacity_hi=float(rng.uniform(0.6, 4.0)))
    w, h = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    tile = int(rng.choice([4, 8, 16, 16, 16, 32]))
    cam = scenes.orbit_camera(azimuth=float(rng.uniform(0, 2 * math.pi)),
                              elevation=float(rng.uniform(-1.2, 1.2)),
                              distance=float(rng.uniform(1.5, 4.0)) * box, width=w, height=h,
                              fov_y=float(rng.uniform(0.3, 1.4)))
    groups = sorted(set(int(g) for g in rng.integers(1, 12, size=int(rng.integers(1, 6)))))
    mask = None if rng.integers(3) == 0 else groups
    return s, cam, tile, mask


@pytest.mark.parametrize("seed", CASES)
def test_fuzz_against_oracle(oracle, seed):
    s, cam, tile, mask = case(seed)
    sub = s if mask is None else filter_scene(s, mask)
    for prec in ("f32", "f64"):
        cfg = RenderConfig(precision=prec, tile_size=tile)
        want = oracle.render_with_state(sub, cam, None, prec, tile_size=tile)
        st = raster.render_with_state(s, cam, mask, config=cfg)
        np.testing.assert_array_equal(st.entries.tile_starts, want.entries.tile_starts)
        assert st.stats.n_drawn == len(want.splats.gids)
        assert st.stats.n_entries == len(want.entries.entry_splat)
        if prec == "f32":
            np.testing.assert_array_equal(st.image, want.image)
            np.testing.assert_array_equal(st.last_contrib, want.last_contrib)
        else:
            assert_image_close(st.image, want.image)
        imgs, cnt = raster.render_views(s, [cam, cam], mask, config=cfg)
        got = imgs[1].cpu().numpy()
        if prec == "f32":
            np.testing.assert_array_equal(got, want.image)
        else:
            assert_image_close(got, want.image)
    fast = raster.render(s, cam, mask, config=RenderConfig(tile_size=tile, exp_mode="fast"))
    want32 = oracle.render_with_state(sub, cam, None, "f32", tile_size=tile).image
    assert_image_close(fast, want32)


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_large_images_against_oracle(oracle, seed):
    """Large and fine tile grids (up to ~140k tiles: the entry-sort fallback of
    render_views, wide radix keys) with dense scenes."""
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([2500, 12000]))
    box = float(rng.uniform(10.0, 25.0))
    s = scenes.random_scene(rng, n, box=box)
    w, h = int(rng.integers(400, 1500)), int(rng.integers(400, 1500))
    tile = int(rng.choice([4, 8, 16, 32] if n < 10000 else [16, 32]))   # E stays < ~30M
    cam = scenes.orbit_camera(azimuth=float(rng.uniform(0, 2 * math.pi)),
                              elevation=float(rng.uniform(-1.0, 1.0)),
                              distance=float(rng.uniform(2.5, 4.0)) * box, width=w, height=h)
    cfg = RenderConfig(tile_size=tile)
    want = oracle.render_with_state(s, cam, None, "f32", tile_size=tile)
    st = raster.render_with_state(s, cam, config=cfg)
    np.testing.assert_array_equal(st.entries.tile_starts, want.entries.tile_starts)
    np.testing.assert_array_equal(st.entries.entry_splat, want.entries.entry_splat)
    np.testing.assert_array_equal(st.image, want.image)
    imgs, cnt = raster.render_views(s, [cam] * 3, config=cfg)
    for k in range(3):
        np.testing.assert_array_equal(imgs[k].cpu().numpy(), want.image)
    fast, _ = raster.render_views(s, [cam], config=RenderConfig(tile_size=tile, exp_mode="fast"))
    assert_image_close(fast[0].cpu().numpy(), want.image)
