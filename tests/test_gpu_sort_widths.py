"""The splat sort's digit width follows the view's depth-code span (g6r_sort.cu
view_key_shape: the fewest <= 9-bit passes, then the narrowest digit that
covers the key -- 3 x 8 bits for the 23-bit codes of the benchmark views).
Scenes built to span a few, a mid and a wide range of f32 depth bits (one
pass up to four), checked bit for bit against the oracle's stable argsort
(raster.py:374-379): tile runs through the exported hot path, and the image."""
import dataclasses

import numpy as np
import pytest

from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.camera import make_camera

from test_gpu_hotpath_runs import hot_runs

pytestmark = pytest.mark.gpu


def _slab_scene(seed, n, depth_extent, distance):
    """n Gaussians in a 30 x 30 slab `depth_extent` deep, `distance` in front
    of a camera on the z axis: the depth codes span ~log2 of the extent's
    share of the depth's f32 ulp."""
    # isotropic: no spatial-directional coupling, so the slab depth is the splat depth
    s = scenes.random_scene(np.random.default_rng(seed), n, box=15.0, iso=True)
    mu_p = s.mu_p.copy()
    mu_p[:, 2] = np.random.default_rng(seed + 1).uniform(-0.5, 0.5, n) * depth_extent
    cam = make_camera((0.0, 0.0, -distance), (0.0, 0.0, 0.0), width=160, height=160, fov_y=0.9)
    return dataclasses.replace(s, mu_p=mu_p), cam


@pytest.mark.parametrize("depth_extent,distance,passes", [
    (1e-4, 40.0, 1),   # 27 distinct depths (5-bit codes): one pass, thousands of ties
    (0.05, 40.0, 2),   # 14-bit codes: two 7-bit passes
    (2.0, 40.0, 3),    # 19-bit codes: three 7-bit passes
    (30.0, 36.0, 3),   # 24-bit codes (an exponent boundary inside): three 8-bit passes
])
def test_splat_sort_runs_bit_exact_across_key_widths(oracle, depth_extent, distance, passes):
    s, cam = _slab_scene(41, 4000, depth_extent, distance)
    want = oracle.render_with_state(s, cam)
    d = want.splats.depths.astype(np.float32).view(np.uint32).astype(np.int64)
    assert len(d) > 100
    bits = int(d.max() - d.min() + 1).bit_length()   # depth codes + the not-drawn code
    assert -(-bits // 9) == passes
    imgs, c, runs = hot_runs(s, [cam, cam])
    for es, ts in runs:
        np.testing.assert_array_equal(ts, want.entries.tile_starts)
        np.testing.assert_array_equal(es, want.entries.entry_splat)
    np.testing.assert_array_equal(imgs[0].cpu().numpy(), want.image)
    # and the image-only path (culled runs) renders the same pixels
    np.testing.assert_array_equal(raster.render_views(s, [cam, cam])[0][1].cpu().numpy(), want.image)
