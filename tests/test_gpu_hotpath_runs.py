"""Bitwise gate on the BENCHMARKED path's sorted runs (SURVEY.md appendix A,
gate 2; reference raster.py:366-379).

``render_views`` -- the throughput path the bench times: chain-free
projection, splat-level depth radix sort, order-preserving tile partition --
never materialises the reference's ``entry_splat`` on its own (the partition
stores scene rows).  With ``entry_splat`` / ``tile_starts`` outputs it maps
rows to compacted SplatBatch indices on the device; these tests require those
runs to equal the reference's bit for bit: against the golden fixtures made by
the unmodified reference, against the oracle at cfg1 / cfg2, in every exp mode
and batch position, and at overflow (empty runs).  The 1M-Gaussian benchmark
scene at 512^2 and 1024^2 is covered in test_gpu_fullsize.py."""

import numpy as np
import pytest
import torch

from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.raster import RenderConfig

from test_oracle import CASES, load_case

pytestmark = pytest.mark.gpu


def hot_runs(scene, cams, config=RenderConfig(), capacity=None):
    """(images, counters, [(entry_splat, tile_starts) per view]) from render_views."""
    prep = raster.prepare_scene(scene, config.w_mode)
    cap = int(capacity or prep.entry_hint)
    tx, ty = raster._tiles(cams[0], int(config.tile_size))
    V = len(cams)
    es = torch.full((V, max(cap, 1)), -7, dtype=torch.int32, device="cuda")
    ts = torch.full((V, tx * ty + 1), -7, dtype=torch.int64, device="cuda")
    imgs, cnt = raster.render_views(scene, cams, config=config, capacity=cap, entry_splat=es,
                                    tile_starts=ts)
    torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    runs = [(es[v, :int(c[v, 1])].cpu().numpy(), ts[v].cpu().numpy()) for v in range(V)]
    return imgs, c, runs


@pytest.mark.parametrize("name", CASES)
def test_hot_path_runs_equal_golden(name):
    z, scene, cam, tile, w_mode = load_case(name)
    for exp in ("exact", "fast"):
        cfg = RenderConfig(precision="f32", w_mode=w_mode, tile_size=tile, exp_mode=exp)
        imgs, c, runs = hot_runs(scene, [cam] * 3, cfg)
        assert int(c[:, 8].sum()) == 0
        for es, ts in runs:
            np.testing.assert_array_equal(ts, z["tile_starts"])
            np.testing.assert_array_equal(es, z["entry_splat"])


def test_hot_path_runs_config1_and_orbit_batch(oracle):
    s = scenes.random_scene(np.random.default_rng(0), 10_000)
    cams = [scenes.benchmark_camera(s, 128, 128)] + scenes.orbit_ring(s, count=12, size=128)[:11]
    _, c, runs = hot_runs(s, cams)
    for cam, (es, ts), cv in zip(cams, runs, c):
        want = oracle.render_with_state(s, cam)
        assert int(cv[0]) == len(want.splats.gids)
        np.testing.assert_array_equal(ts, want.entries.tile_starts)
        np.testing.assert_array_equal(es, want.entries.entry_splat)


def test_hot_path_runs_config2_200k_512(oracle):
    s = scenes.phantom_agp_scene((128, 128, 128)).take(np.arange(200_000))
    cam = scenes.benchmark_camera(s, 512, 512)
    want = oracle.render_with_state(s, cam)
    imgs, c, runs = hot_runs(s, [cam, cam])
    for es, ts in runs:
        np.testing.assert_array_equal(ts, want.entries.tile_starts)
        np.testing.assert_array_equal(es, want.entries.entry_splat)
    np.testing.assert_array_equal(imgs[1].cpu().numpy(), want.image)


def test_hot_path_runs_group_mask_and_tiles(oracle):
    s = scenes.random_scene(np.random.default_rng(5), 6000)
    cam = scenes.orbit_ring(s, count=8, size=200)[3]
    for tile in (8, 16, 32):
        for mask in (None, (2, 5), (7,)):
            cfg = RenderConfig(tile_size=tile)
            want = oracle.render_with_state(s, cam, mask, tile_size=tile)
            prep = raster.prepare_scene(s)
            tx, ty = raster._tiles(cam, tile)
            es = torch.empty((1, prep.entry_hint), dtype=torch.int32, device="cuda")
            ts = torch.empty((1, tx * ty + 1), dtype=torch.int64, device="cuda")
            _, cnt = raster.render_views(s, [cam], group_mask=mask, config=cfg, entry_splat=es,
                                         tile_starts=ts)
            e = int(cnt[0, 1].item())
            np.testing.assert_array_equal(ts[0].cpu().numpy(), want.entries.tile_starts)
            np.testing.assert_array_equal(es[0, :e].cpu().numpy(), want.entries.entry_splat)


def test_hot_path_runs_overflow_gives_empty_runs():
    s = scenes.random_scene(np.random.default_rng(3), 3000)
    cam = scenes.orbit_ring(s, count=4, size=128)[1]
    imgs, c, runs = hot_runs(s, [cam], capacity=16)
    assert int(c[0, 8]) == 1
    es, ts = runs[0]
    assert (ts == 0).all()


def test_hot_path_runs_only_for_views_that_ask():
    """Frames without entry_splat in the same batch are untouched and the
    images are unchanged by the export."""
    s = scenes.random_scene(np.random.default_rng(11), 4000)
    cams = scenes.orbit_ring(s, count=6, size=96)
    a, ca = raster.render_views(s, cams)
    b, cb, runs = hot_runs(s, cams)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(ca, torch.from_numpy(cb).cuda())
    for cam, (es, ts) in zip(cams, runs):
        st = raster.render_with_state(s, cam)
        np.testing.assert_array_equal(es, st.entries.entry_splat)
        np.testing.assert_array_equal(ts, st.entries.tile_starts)
