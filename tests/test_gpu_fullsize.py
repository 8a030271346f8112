"""Parity at the benchmark's own sizes (BASELINE.json configs[2] and [3]): the
1M-Gaussian Psi-decoded scene, one orbit view at 512x512 and one at 1024x1024,
rendered on the device and by the CPU oracle (which is pinned bit-for-bit to the
reference by test_oracle.py).  Tile runs and the f32 framebuffer are compared
bit for bit through both device paths -- render_with_state (ordered projection,
entry sort) and render_views (chain-free projection, splat-level sort, tile
partition) -- and the fast-exp mode against the parity bound."""
import numpy as np
import pytest
import torch

from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig

from test_gpu_hotpath_runs import hot_runs
from test_gpu_parity import assert_image_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene1m():
    return scenes.psi_decode_scene(352, limit=1_000_000)


@pytest.mark.parametrize("size,count,view", [(512, 100, 7), (1024, 800, 300)])
def test_full_size_view_matches_oracle(oracle, scene1m, size, count, view):
    cam = scenes.orbit_ring(scene1m, count=count, size=size)[view]
    want = oracle.render_with_state(scene1m, cam)
    st = raster.render_with_state(scene1m, cam)
    assert st.stats.n_drawn > 900_000 and st.stats.n_entries > 1_500_000
    np.testing.assert_array_equal(st.splats.gids, want.splats.gids)
    np.testing.assert_array_equal(st.entries.tile_starts, want.entries.tile_starts)
    np.testing.assert_array_equal(st.entries.entry_splat, want.entries.entry_splat)
    np.testing.assert_array_equal(st.image, want.image)
    np.testing.assert_array_equal(st.last_contrib, want.last_contrib)
    np.testing.assert_array_equal(st.final_t, want.final_t)
    # the benchmarked path: splat sort + tile partition, runs exported
    imgs, c, runs = hot_runs(scene1m, [cam, cam])
    assert int(c[:, 8].sum()) == 0
    assert tuple(c[0, :2]) == (st.stats.n_drawn, st.stats.n_entries)
    for k in range(2):
        np.testing.assert_array_equal(runs[k][1], want.entries.tile_starts)
        np.testing.assert_array_equal(runs[k][0], want.entries.entry_splat)
        np.testing.assert_array_equal(imgs[k].cpu().numpy(), want.image)
    fast, _ = raster.render_views(scene1m, [cam], config=RenderConfig(exp_mode="fast"))
    assert_image_close(fast[0].cpu().numpy(), want.image)
