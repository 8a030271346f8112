"""Parity of the CUDA render path with the CPU oracle and the reference's
golden vectors (needs a B200: ``-m gpu``).

Gates:
  * prep: device terms vs oracle within a few ulp (transcendentals differ in
    the last bit between CUDA and numpy's SIMD exp/tanh; everything else is
    IEEE basic ops in the reference's order);
  * projection: given the oracle's prep, means2d/conics/colors/depths/radii
    and the kept set bit-identical, alphas within 1 ulp;
  * binning: given the oracle's splats, entry_splat and tile_starts bit-exact;
  * end to end: tile runs bit-exact, f32 and f64 images within max-abs 1e-3 /
    PSNR >= 60 dB (and reported bitwise fractions; f32 is expected bitwise);
  * masks byte-identical to pre-filtered scenes, determinism, the degenerate
    policy, and the reference's kernel hand cases through the adapter.
"""

import glob
import math
import os
import threading

import numpy as np
import pytest

from paper_2505_17338_b200 import kernels as K
from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.errors import DegenerateCovarianceError
from paper_2505_17338_b200.raster import RenderConfig, SplatBatch
from paper_2505_17338_b200.scene import filter_scene

from test_oracle import CASES, GOLDEN, load_case

pytestmark = pytest.mark.gpu
F64 = RenderConfig(precision="f64")


def ulp_diff(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.spacing(np.maximum(np.abs(a), np.abs(b))), 1e-300)


def psnr(a, b):
    d = np.asarray(a, np.float64)[..., :3] - np.asarray(b, np.float64)[..., :3]
    mse = float(np.mean(d * d))
    return math.inf if mse == 0 else 10 * math.log10(1.0 / mse)


def assert_image_close(got, want):
    assert got.shape == want.shape and got.dtype == want.dtype
    diff = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert diff.max() <= 1e-3, diff.max()
    assert psnr(got, want) >= 60.0


# --- device expf --------------------------------------------------------------

def test_device_expf_is_glibc_on_every_float_in_the_compositor_range(oracle):
    import ctypes
    import torch
    from paper_2505_17338_b200 import _native as nat
    lo = np.float32(-4.5).view(np.uint32)
    # all floats in [-4.5, -0.0]: bit patterns 0x80000000 .. bits(-4.5)
    bits = np.arange(0x80000000, int(lo) + 1, dtype=np.uint64).astype(np.uint32)
    x = torch.from_numpy(bits.view(np.float32)).cuda()
    y = torch.empty_like(x)
    nat.check(nat.load().g6r_debug_expf(x.numel(), ctypes.c_void_p(x.data_ptr()),
                                        ctypes.c_void_p(y.data_ptr()), raster._stream_handle()))
    got = y.cpu().numpy()
    idx = np.random.default_rng(0).choice(len(bits), 2_000_000, replace=False)
    np.testing.assert_array_equal(got[idx], oracle.expf_glibc(bits[idx].view(np.float32)))
    z = np.load(os.path.join(GOLDEN, "expf_glibc.npz"))
    xs = torch.from_numpy(z["x"]).cuda()
    ys = torch.empty_like(xs)
    nat.check(nat.load().g6r_debug_expf(xs.numel(), ctypes.c_void_p(xs.data_ptr()),
                                        ctypes.c_void_p(ys.data_ptr()), raster._stream_handle()))
    np.testing.assert_array_equal(ys.cpu().numpy(), z["y"])


# --- golden fixtures end to end ---------------------------------------------------

@pytest.mark.parametrize("name", CASES)
def test_golden_end_to_end(name):
    z, scene, cam, tile, w_mode = load_case(name)
    for prec in ("f32", "f64"):
        cfg = RenderConfig(precision=prec, w_mode=w_mode, tile_size=tile)
        st = raster.render_with_state(scene, cam, config=cfg)
        np.testing.assert_array_equal(st.entries.tile_starts, z["tile_starts"])
        np.testing.assert_array_equal(st.entries.entry_splat, z["entry_splat"])
        np.testing.assert_array_equal(st.splats.gids, z["splat_gids"])
        np.testing.assert_array_equal(st.splats.radii, z["splat_radii"])
        # f64 means: prep transcendentals (exp, tanh) may differ from numpy in the
        # last ulp and the slicing amplifies that a little; 1e-9 px is ~1e4x below
        # what could move a pixel-centre test
        assert np.abs(st.splats.means2d - z["splat_means2d"]).max() <= 1e-9
        assert_image_close(st.image, z[f"{prec}_image"])
        if prec == "f32":
            np.testing.assert_array_equal(st.image, z["f32_image"])
            np.testing.assert_array_equal(st.last_contrib, z["f32_last_contrib"])
        stats = z["stats"]
        assert (st.stats.n_drawn, st.stats.n_entries) == (stats[0], stats[1])
        assert (st.stats.n_view_degenerate, st.stats.n_alpha_culled, st.stats.n_depth_culled,
                st.stats.n_projection_culled, st.stats.n_viewport_culled) == tuple(stats[2:7])


@pytest.mark.parametrize("name", CASES)
def test_golden_hot_path(name):
    """The throughput path (chain-free projection: entries in CTA-completion
    order, equal keys put back in row order after the sort) gives the golden
    f32 image bit for bit -- incl. `ties50`, whose equal depths make the tie
    rule visible in the compositing order."""
    z, scene, cam, tile, w_mode = load_case(name)
    cfg = RenderConfig(precision="f32", w_mode=w_mode, tile_size=tile)
    imgs, counters = raster.render_views(scene, [cam] * 3, config=cfg)
    c = counters.cpu().numpy()
    assert int(c[:, 8].sum()) == 0
    assert tuple(c[0, :2]) == tuple(z["stats"][:2])
    for k in range(3):
        np.testing.assert_array_equal(imgs[k].cpu().numpy(), z["f32_image"])
    np.testing.assert_array_equal(raster.render(scene, cam, config=cfg), z["f32_image"])


def test_pipelined_batches_match_unpipelined():
    """19 views = three batches on the two pipelined streams vs one stream."""
    s = scenes.random_scene(np.random.default_rng(72), 20000)
    cams = scenes.orbit_ring(s, count=19, size=128)
    a, ca = raster.render_views(s, cams)
    b, cb = raster.render_views(s, cams, pipeline=False)
    import torch
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(ca, cb)
    host = raster.render_batch(s, cams)
    np.testing.assert_array_equal(host, a.cpu().numpy())


# --- stage gates ------------------------------------------------------------------

@pytest.mark.parametrize("seed,n,w_mode", [(21, 3000, "peak"), (22, 3000, "raw")])
def test_prep_terms_match_oracle(oracle, seed, n, w_mode):
    s = scenes.random_scene(np.random.default_rng(seed), n)
    want = oracle.prepare(s, w_mode)
    got = raster.prepare_scene(s, w_mode)
    np.testing.assert_array_equal(got.terms.degenerate, want.degenerate)
    for f in ("adjust", "precision_dd", "sigma_prime", "w_norm"):
        a, b = getattr(got.terms, f), getattr(want, f)
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14 * np.abs(b).max(), err_msg=f)
    assert ulp_diff(got.opacity, want.opacity).max() <= 2


@pytest.mark.parametrize("seed,n", [(31, 4000), (32, 20000)])
def test_projection_bitwise_given_oracle_prep(oracle, seed, n):
    s = scenes.random_scene(np.random.default_rng(seed), n)
    cam = scenes.orbit_camera(azimuth=0.3, elevation=-0.2, width=160, height=128)
    op = oracle.prepare(s)
    prep = raster.prepare_from_terms(s, op, op.opacity)
    stats = raster.RenderStats()
    got = raster.project_scene(s, prep, np.arange(n), cam, RenderConfig(), stats)
    rows, _, _ = oracle.select_rows(s, op, None)
    want = oracle.project(s, op, rows, cam)
    np.testing.assert_array_equal(got.gids, want.gids)
    for f in ("means2d", "conics", "colors", "depths", "radii"):
        np.testing.assert_array_equal(getattr(got, f), getattr(want, f), err_msg=f)
    # exp(-q/2): CUDA exp and numpy's SIMD exp are each within 1 ulp of exact
    assert ulp_diff(got.alphas, want.alphas).max() <= 2
    np.testing.assert_array_equal(np.bincount(want.stage, minlength=6)[1:6],
                                  [stats.n_view_degenerate, stats.n_alpha_culled,
                                   stats.n_depth_culled, stats.n_projection_culled,
                                   stats.n_viewport_culled])


@pytest.mark.parametrize("tile", [16, 8, 5])
def test_binning_bitwise_given_oracle_splats(oracle, tile):
    s = scenes.random_scene(np.random.default_rng(41), 30000)
    cam = scenes.orbit_camera(azimuth=1.0, elevation=0.3, width=250, height=190)
    st = oracle.render_with_state(s, cam, tile_size=tile)
    sp = st.splats
    got = raster.bin_splats(SplatBatch(sp.gids, sp.means2d, sp.conics, sp.colors, sp.alphas,
                                       sp.depths, sp.radii), cam, tile)
    np.testing.assert_array_equal(got.tile_starts, st.entries.tile_starts)
    np.testing.assert_array_equal(got.entry_splat, st.entries.entry_splat)


def test_composite_bitwise_given_oracle_runs(oracle):
    s = scenes.random_scene(np.random.default_rng(43), 20000)
    cam = scenes.orbit_camera(azimuth=-0.5, elevation=0.1, width=200, height=200)
    for prec in ("f32", "f64"):
        st = oracle.render_with_state(s, cam, precision=prec)
        sp = SplatBatch(st.splats.gids, st.splats.means2d, st.splats.conics, st.splats.colors,
                        st.splats.alphas, st.splats.depths, st.splats.radii)
        en = raster.TileEntries(st.entries.entry_splat, st.entries.tile_starts,
                                st.entries.tiles_x, st.entries.tiles_y)
        img, ft, last = raster.composite_splats(sp, en, cam, RenderConfig(precision=prec))
        # both precisions bit for bit: f32 through the restated glibc expf,
        # f64 through the restated glibc exp (the oracle calls the host libm)
        np.testing.assert_array_equal(img, st.image)
        np.testing.assert_array_equal(ft, st.final_t)
        np.testing.assert_array_equal(last, st.last_contrib)


def test_device_exp_is_glibc(oracle):
    """The f64 compositors' exp equals the host libm's on 24M doubles: the
    compositor range [-4.5, 0] (uniform and a dense grid), the restatement's
    whole domain (-512, 512) and tiny arguments."""
    import ctypes
    import torch
    from paper_2505_17338_b200 import _native as nat
    rng = np.random.default_rng(5)
    xs = np.concatenate([-4.5 * rng.random(8_000_000), np.linspace(-4.5, 0.0, 8_000_001),
                         rng.uniform(-511.9, 511.9, 8_000_000),
                         np.array([0.0, -0.0, 1e-300, -1e-300, 2.0 ** -60, -(2.0 ** -54), 2.0 ** -54])])
    x = torch.from_numpy(xs).cuda()
    y = torch.empty_like(x)
    nat.check(nat.load().g6r_debug_exp(x.numel(), ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr()), raster._stream_handle()))
    got = y.cpu().numpy()
    want = np.array([math.exp(v) for v in xs[::97]])
    np.testing.assert_array_equal(got[::97], want)
    # the full set against numpy's scalar-path equivalent (math.exp per value is slow):
    # vectorised libm through the oracle's C library
    np.testing.assert_array_equal(got, oracle.libm_exp(xs))


def test_f64_render_bit_identical_to_brute_force_rule(oracle):
    """render_with_state(f64) composites its own splats exactly like the
    reference kernel (libm exp, same order): bit for bit against the oracle's
    f64 compositor on the same runs (the reference's own test_raster.py:414-457
    pins this against a brute-force loop; tests/test_gpu_integrate.py runs it)."""
    for seed, n in ((0, 1), (1, 10), (2, 40), (3, 100), (4, 3000)):
        s = scenes.random_scene(np.random.default_rng(seed), n)
        cam = scenes.orbit_camera(azimuth=0.3 * seed, elevation=0.15 * seed, width=48, height=40)
        st = raster.render_with_state(s, cam, config=F64)
        img, ft, last = oracle.composite(st.splats.means2d, st.splats.conics, st.splats.colors,
                                         st.splats.alphas, st.entries.entry_splat,
                                         st.entries.tile_starts, st.entries.tiles_x, 16,
                                         cam.width, cam.height, "f64")
        np.testing.assert_array_equal(st.image, img)
        np.testing.assert_array_equal(st.final_t, ft)
        np.testing.assert_array_equal(st.last_contrib, last)


# --- end to end at configuration sizes -----------------------------------------------

def test_config1_10k_random_128(oracle):
    s = scenes.random_scene(np.random.default_rng(0), 10_000)
    cam = scenes.benchmark_camera(s, 128, 128)
    for prec in ("f32", "f64"):
        st = raster.render_with_state(s, cam, config=RenderConfig(precision=prec))
        want = oracle.render_with_state(s, cam, precision=prec)
        np.testing.assert_array_equal(st.entries.tile_starts, want.entries.tile_starts)
        np.testing.assert_array_equal(st.entries.entry_splat, want.entries.entry_splat)
        assert_image_close(st.image, want.image)
    assert st.stats.n_entries > 50_000


def test_config2_200k_phantom_512(oracle):
    s = scenes.phantom_agp_scene((128, 128, 128)).take(np.arange(200_000))
    cam = scenes.benchmark_camera(s, 512, 512)
    st = raster.render_with_state(s, cam)
    want = oracle.render_with_state(s, cam)
    np.testing.assert_array_equal(st.splats.gids, want.splats.gids)
    np.testing.assert_array_equal(st.entries.tile_starts, want.entries.tile_starts)
    np.testing.assert_array_equal(st.entries.entry_splat, want.entries.entry_splat)
    assert_image_close(st.image, want.image)
    np.testing.assert_array_equal(st.image, want.image)


# --- policies, masks, determinism ------------------------------------------------------

@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_group_mask_equals_prefiltered_scene(precision):
    s = scenes.random_scene(np.random.default_rng(47), 900)
    cam = scenes.orbit_camera(azimuth=2.0, elevation=-0.2, width=96, height=96)
    cfg = RenderConfig(precision=precision)
    for groups in ([7], [2, 5], [5, 7], [2, 5, 7], list(range(1, 12))):
        masked = raster.render(s, cam, group_mask=groups, config=cfg)
        filtered = raster.render(filter_scene(s, groups), cam, config=cfg)
        np.testing.assert_array_equal(masked, filtered)


def test_all_masked_gives_transparent_black():
    s = scenes.random_scene(np.random.default_rng(59), 20)
    s = s.with_params(labels=np.full(20, 4, dtype=np.uint8))
    img = raster.render(s, scenes.orbit_camera(), group_mask=[7])
    assert img.shape == (64, 64, 4) and np.all(img == 0.0)


def test_determinism_repeat_and_concurrent():
    s = scenes.random_scene(np.random.default_rng(61), 5000)
    cam = scenes.orbit_camera(azimuth=0.9, width=128, height=96)
    base = raster.render(s, cam)
    np.testing.assert_array_equal(raster.render(s, cam), base)
    out = [None] * 8

    def work(i):
        import torch
        with torch.cuda.stream(torch.cuda.Stream()):
            out[i] = raster.render(s, cam)

    th = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    [t.start() for t in th]
    [t.join() for t in th]
    for o in out:
        np.testing.assert_array_equal(o, base)


def test_concurrent_pipelined_batches_from_threads():
    """Several host threads render pipelined multi-batch calls on their own
    streams at once (the library's internal lane streams are shared): every
    result equals the single-threaded one."""
    import torch
    s = scenes.random_scene(np.random.default_rng(62), 20000)
    cams = scenes.orbit_ring(s, count=20, size=96)
    base = raster.render_batch(s, cams)
    out = [None] * 4

    def work(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            imgs, _ = raster.render_views(s, cams)
            out[i] = imgs.cpu().numpy()

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    for o in out:
        np.testing.assert_array_equal(o, base)


def test_degenerate_policy_on_device():
    s = scenes.random_scene(np.random.default_rng(83), 300)
    cov = s.cov_raw.copy()
    cov[:2, 3:6] = -300.0
    cov[:2, 9:] = 0.0
    s2 = s.with_params(cov_raw=cov)
    st = raster.render_with_state(s2, scenes.orbit_camera(), config=F64)
    assert st.stats.n_degenerate == 2
    clean = s2.take(np.arange(2, 300))
    np.testing.assert_array_equal(st.image, raster.render(clean, scenes.orbit_camera(), config=F64))
    cov[:5, 3:6] = -300.0
    cov[:5, 9:] = 0.0
    with pytest.raises(DegenerateCovarianceError):
        raster.render(s.with_params(cov_raw=cov), scenes.orbit_camera(), config=F64)


def test_entry_overflow_rerenders_transparently():
    s = scenes.random_scene(np.random.default_rng(67), 3000)
    cam = scenes.orbit_camera(width=128, height=128)
    want = raster.render(s, cam)
    prep = raster.prepare_scene(s)
    prep.entry_hint = 100   # far too small: device reports overflow, host re-renders
    np.testing.assert_array_equal(raster.render(s, cam), want)
    assert prep.entry_hint > 100


def test_render_views_matches_single_views():
    s = scenes.random_scene(np.random.default_rng(71), 4000)
    cams = scenes.orbit_ring(s, count=6, size=96)
    imgs, counters = raster.render_views(s, cams)
    assert int(counters[:, 8].sum()) == 0
    for k, cam in enumerate(cams):
        np.testing.assert_array_equal(imgs[k].cpu().numpy(), raster.render(s, cam))


# --- reference kernel hand cases through the kernel-module adapter ----------------------

def composite_direct(dtype, means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
                     tile_size, height, width):
    image = np.zeros((height, width, 4), dtype=dtype)
    final_t = np.ones((height, width), dtype=dtype)
    last = np.zeros((height, width), dtype=np.int32)
    K.composite_forward(np.asarray(means2d, dtype), np.asarray(conics, dtype),
                        np.asarray(colors, dtype), np.asarray(alphas, dtype),
                        np.asarray(entry_splat, np.int32), np.asarray(tile_starts, np.int64),
                        tiles_x, tile_size, image, final_t, last, 1)
    return image, final_t, last


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_kernel_hand_cases(dtype):
    img, ft, last = composite_direct(dtype, [[8.0, 8.0]], [[0.1, 0.0, 0.1]], [[1.0, 0.0, 0.0]],
                                     [0.9], [0], [0, 1], 1, 16, 16, 16)
    np.testing.assert_array_equal(img[8, 8], np.array([0.9, 0.0, 0.0, 0.9], dtype))
    assert last[8, 8] == 1 and ft[8, 8] == pytest.approx(0.1, rel=1e-6)
    img, _, _ = composite_direct(dtype, [[8.0, 8.0]] * 2, [[0.1, 0.0, 0.1]] * 2,
                                 [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]], [0.6, 0.5], [0, 1], [0, 2], 1,
                                 16, 16, 16)
    np.testing.assert_allclose(img[8, 8], [0.6, 0.5 * 0.4, 0.0, 0.6 + 0.5 * 0.4], atol=1e-7)
    img, _, _ = composite_direct(dtype, [[0.0, 0.0]], [[-0.5, 0.0, -0.5]], [[1.0, 1.0, 1.0]],
                                 [0.9], [0], [0, 1], 1, 16, 16, 16)
    assert img[0, 0, 3] == dtype(0.9) and np.all(img[1:, 1:, 3] == 0.0)
    img, _, _ = composite_direct(dtype, [[0.0, 0.0]], [[1.0, 0.0, 1.0]], [[1.0, 1.0, 1.0]], [0.9],
                                 [0], [0, 1], 1, 16, 1, 16)
    assert img[0, 3, 3] == pytest.approx(0.9 * math.exp(-4.5), rel=1e-6)
    assert np.all(img[0, 4:, 3] == 0.0)
    img, _, last = composite_direct(dtype, [[8.0, 8.0]], [[0.1, 0.0, 0.1]], [[1.0, 1.0, 1.0]],
                                    [0.003], [0], [0, 1], 1, 16, 16, 16)
    assert np.all(img == 0.0) and np.all(last == 0)
    img, ft, last = composite_direct(dtype, [[8.0, 8.0]] * 3, [[1e-6, 0.0, 1e-6]] * 3,
                                     [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]],
                                     [0.999] * 3, [0, 1, 2], [0, 3], 1, 16, 16, 16)
    assert last[8, 8] == 2 and img[8, 8, 2] == 0.0
    assert ft[8, 8] == pytest.approx(1e-6, rel=1e-3)
    img, ft, last = composite_direct(dtype, np.zeros((0, 2)), np.zeros((0, 3)), np.zeros((0, 3)),
                                     np.zeros(0), np.zeros(0), [0, 0], 1, 16, 16, 16)
    assert np.all(img == 0.0) and np.all(ft == 1.0) and np.all(last == 0)


def test_kernel_module_projection_stages_match_oracle(oracle):
    s = scenes.random_scene(np.random.default_rng(91), 2000)
    cam = scenes.orbit_camera(azimuth=0.2, width=96, height=96)
    op = oracle.prepare(s)
    n = len(s)
    pos = cam.position
    got, want = {}, {}
    for mod, out in ((K, got), (oracle.lib(), want)):
        stage = np.zeros(n, np.uint8)
        view, madj, quad = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n)
        if mod is K:
            K.project_stage1(s.mu_p, s.mu_d, op.adjust, op.precision_dd, *pos, view, madj, quad, stage)
        else:
            mod.or_project_stage1(n, *[oracle._p(np.ascontiguousarray(a)) for a in
                                       (s.mu_p, s.mu_d, op.adjust, op.precision_dd)], *pos,
                                  oracle._p(view), oracle._p(madj), oracle._p(quad), oracle._p(stage))
        out.update(view=view, madj=madj, quad=quad, stage=stage)
    for k in got:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)


BWD_CASES = ("rand40", "rand400", "rand400_raw", "cull100", "rand1500_wide", "rand2000_low", "rand800_raw")


@pytest.mark.parametrize("name", BWD_CASES)
def test_render_backward_matches_reference_golden(name):
    """Full backward (compositor adjoint + per-splat chain to all 40 raw
    parameters) vs the reference's render_backward on the golden scenes.
    Tolerance: pixel sums are associated differently (deterministic tree
    instead of sequential) and prep transcendentals differ in the last ulp."""
    from paper_2505_17338_b200.diffrender import render_backward
    z, scene, cam, tile, w_mode = load_case(name)
    zb = np.load(os.path.join(GOLDEN, f"bwd_{name}.npz"))
    got = render_backward(scene, cam, zb["grad_image"], config=RenderConfig(w_mode=w_mode))
    for f in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw"):
        want = zb[f"g_{f}"]
        scale = max(float(np.abs(want).max()), 1e-30)
        np.testing.assert_allclose(getattr(got, f), want, rtol=1e-7, atol=1e-9 * scale, err_msg=f)
    assert got.all_finite()


def test_render_backward_deterministic_and_zero_for_culled():
    from paper_2505_17338_b200.diffrender import render_backward
    z, scene, cam, tile, w_mode = load_case("cull100")
    zb = np.load(os.path.join(GOLDEN, "bwd_cull100.npz"))
    a = render_backward(scene, cam, zb["grad_image"])
    b = render_backward(scene, cam, zb["grad_image"])
    for f in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    drawn = np.zeros(len(scene), dtype=bool)
    drawn[z["splat_gids"]] = True
    assert np.all(a.cov_raw[~drawn] == 0.0) and np.all(a.opacity_raw[~drawn] == 0.0)


def oracle_accumulate(oracle, s, en, st, g, init):
    """The oracle's composite_backward into rows pre-filled with `init` (+=)."""
    return oracle.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat,
                                     en.tile_starts, en.tiles_x, 16, st.final_t.shape[1],
                                     st.final_t.shape[0], st.final_t, st.last_contrib, g,
                                     init=init)


def test_backward_matches_oracle(oracle):
    z, scene, cam, tile, w_mode = load_case("rand400")
    st = oracle.render_with_state(scene, cam, None, "f64")
    s, en = st.splats, st.entries
    g = np.random.default_rng(2).normal(size=st.image.shape)
    want = oracle.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat,
                                     en.tile_starts, en.tiles_x, 16, cam.width, cam.height,
                                     st.final_t, st.last_contrib, g)
    got = np.zeros_like(want)
    K.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat, en.tile_starts,
                         en.tiles_x, 16, st.final_t, st.last_contrib, g, got)
    # deterministic (no float atomics): the reference's summation order, bit for bit
    np.testing.assert_array_equal(got, want)
    again = np.full_like(want, 0.25)
    K.composite_backward(s.means2d, s.conics, s.colors, s.alphas, en.entry_splat, en.tile_starts,
                         en.tiles_x, 16, st.final_t, st.last_contrib, g, again)
    np.testing.assert_array_equal(again, oracle_accumulate(oracle, s, en, st, g, 0.25))


# --- edge cases of the reference's input domain ---------------------------------------

@pytest.mark.parametrize("size", [(1, 1), (17, 13), (16, 16), (33, 7)])
@pytest.mark.parametrize("tile", [16, 8, 32])
def test_odd_image_and_tile_sizes_match_oracle(oracle, size, tile):
    s = scenes.random_scene(np.random.default_rng(size[0] * 7 + tile), 600, box=6.0)
    cam = scenes.orbit_camera(azimuth=0.4, elevation=0.1, distance=25.0, width=size[0],
                              height=size[1])
    for prec in ("f32", "f64"):
        cfg = RenderConfig(precision=prec, tile_size=tile)
        want = oracle.render_with_state(s, cam, None, prec, tile_size=tile)
        got = raster.render(s, cam, config=cfg)
        if prec == "f32":
            np.testing.assert_array_equal(got, want.image)
        else:
            assert_image_close(got, want.image)
        imgs, _ = raster.render_views(s, [cam, cam], config=cfg)
        np.testing.assert_array_equal(imgs[1].cpu().numpy(), got)


def test_empty_scene_and_nothing_visible():
    from paper_2505_17338_b200.scene import Scene
    empty = Scene(mu_p=np.zeros((0, 3)), mu_d=np.zeros((0, 3)), cov_raw=np.zeros((0, 21)),
                  sh=np.zeros((0, 12)), opacity_raw=np.zeros(0), labels=np.zeros(0, np.uint8))
    cam = scenes.orbit_camera(width=40, height=24)
    assert not raster.render(empty, cam).any()
    st = raster.render_with_state(empty, cam)
    assert st.stats.n_drawn == 0 and len(st.entries.entry_splat) == 0
    assert not raster.render_frames_u8(empty, [cam], (1.0, 0.0, 0.0))[0][:, :, 1].any()
    # a scene entirely behind the camera
    s = scenes.random_scene(np.random.default_rng(3), 200, box=2.0)
    behind = scenes.orbit_camera(azimuth=0.0, distance=70.0, width=32, height=32,
                                 target=(0.0, 0.0, -200.0))   # looks away from the scene
    img = raster.render(s, behind)
    assert not img.any()


def test_f64_batched_views_match_single_renders():
    s = scenes.random_scene(np.random.default_rng(81), 3000)
    cams = scenes.orbit_ring(s, count=10, size=64)
    cfg = RenderConfig(precision="f64")
    imgs, _ = raster.render_views(s, cams, config=cfg)
    for k, cam in enumerate(cams):
        np.testing.assert_array_equal(imgs[k].cpu().numpy(), raster.render(s, cam, config=cfg))


def test_splat_sort_windows_and_large_grids_match_entry_sort(oracle):
    """Hot path (splat-level sort) vs the entry sort (render_with_state) on a
    scene with a few huge splats -- rounds whose entries span several 4096-entry
    windows -- at 1024x1024 (4096 tiles, splat sort) and at 1040x1040 (4225
    tiles, entry sort for both)."""
    s = scenes.random_scene(np.random.default_rng(91), 3000, box=10.0)
    big = np.argsort(s.mu_p[:, 2])[:6]          # enlarge a few Gaussians a lot
    cov = s.cov_raw.copy()
    cov[big, :3] += 4.0   # each covers the whole image: > 4096 entries in its round
    from dataclasses import replace
    s = replace(s, cov_raw=cov)
    for size in (1024, 1040):
        cam = scenes.orbit_camera(azimuth=0.2, elevation=0.1, distance=40.0, width=size, height=size)
        st = raster.render_with_state(s, cam)
        hot = raster.render(s, cam)
        np.testing.assert_array_equal(hot, st.image)
        imgs, cnt = raster.render_views(s, [cam, cam])
        np.testing.assert_array_equal(imgs[0].cpu().numpy(), st.image)
        assert int(cnt[0, 1]) == st.stats.n_entries
    ref = oracle.render_with_state(s, scenes.orbit_camera(azimuth=0.2, elevation=0.1, distance=40.0,
                                                          width=1024, height=1024))
    np.testing.assert_array_equal(raster.render(s, scenes.orbit_camera(
        azimuth=0.2, elevation=0.1, distance=40.0, width=1024, height=1024)), ref.image)
