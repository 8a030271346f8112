"""Served-frame output path: the fused composite-over +
8-bit quantisation epilogue against the reference's host formula
(metrics.py:21-25 composite_over, _png.py:21-32 to_rgba_u8) applied to the
oracle's image, byte for byte, and the PNG container against PIL on the same
pixels."""

import io

import numpy as np
import pytest

from paper_2505_17338_b200 import output, raster, scenes
from paper_2505_17338_b200.raster import RenderConfig

pytestmark = pytest.mark.gpu


def reference_rgba8(image, bg):
    """to_rgba_u8(composite_over(image, bg)), restated (numpy, f64)."""
    img = np.asarray(image, np.float64)
    rgb = img[:, :, :3] + np.asarray(bg, np.float64) * (1.0 - img[:, :, 3:4])
    arr = np.concatenate([rgb, np.ones_like(rgb[:, :, :1])], axis=2)
    return np.round(np.clip(arr, 0.0, 1.0) * 255.0).astype(np.uint8)


@pytest.mark.parametrize("bg", [(0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (0.2, 0.5, 0.9)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_fused_frames_match_reference_quantisation(oracle, bg, prec):
    s = scenes.random_scene(np.random.default_rng(3), 3000)
    cams = [scenes.orbit_camera(azimuth=a, elevation=0.2, width=96, height=72) for a in (0.0, 1.1, 2.5)]
    cfg = RenderConfig(precision=prec)
    got = raster.render_frames_u8(s, cams, bg, config=cfg)
    assert got.shape == (3, 72, 96, 4) and got.dtype == np.uint8
    for v, cam in enumerate(cams):
        want = reference_rgba8(oracle.render(s, cam, precision=prec), bg)
        np.testing.assert_array_equal(got[v], want)
        # and identical to quantising the device's own float image
        np.testing.assert_array_equal(got[v], reference_rgba8(raster.render(s, cam, config=cfg), bg))


def test_frames_with_masks_and_many_views_match_float_path():
    s = scenes.random_scene(np.random.default_rng(4), 20000)
    cams = [scenes.orbit_camera(azimuth=0.3 * k, width=128, height=128) for k in range(11)]
    imgs = raster.render_batch(s, cams, group_mask=[1, 4, 6])
    got = raster.render_frames_u8(s, cams, (0.1, 0.1, 0.1), group_mask=[1, 4, 6])
    for v in range(len(cams)):
        np.testing.assert_array_equal(got[v], reference_rgba8(imgs[v], (0.1, 0.1, 0.1)))


def test_png_bytes_match_reference_encoding():
    from PIL import Image
    s = scenes.random_scene(np.random.default_rng(5), 2000)
    cam = scenes.orbit_camera(azimuth=0.7, width=80, height=64)
    data = output.render_png(s, cam, background=(0.0, 0.0, 0.0))
    want = reference_rgba8(raster.render(s, cam), (0.0, 0.0, 0.0))
    buf = io.BytesIO()
    Image.fromarray(want, mode="RGBA").save(buf, format="PNG", compress_level=6)
    assert data == buf.getvalue()
    with Image.open(io.BytesIO(data)) as im:
        np.testing.assert_array_equal(np.asarray(im.convert("RGBA")), want)
