"""Host-side logic of the drop-in (CPU-only): config validation, group masks,
the degenerate policy, input contracts, view sharding, scene synthesis, and
the C ABI surface of libg6r.so (loaded without a GPU; no compute calls)."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from paper_2505_17338_b200 import _native as nat
from paper_2505_17338_b200 import multigpu, raster, scenes
from paper_2505_17338_b200.camera import Camera, make_camera
from paper_2505_17338_b200.errors import (DegenerateCovarianceError, DegenerateGeometryError,
                                          InvalidParameterError)
from paper_2505_17338_b200.scene import Scene, filter_scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# --- C ABI ----------------------------------------------------------------

def header_symbols():
    text = open(os.path.join(ROOT, "include", "g6r.h")).read()
    return sorted(set(re.findall(r"\b(g6r_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = nat.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
        assert name in nat.EXPORTED, f"{name} has no ctypes signature"
    assert "sm_100a" in nat.version()


def test_frame_struct_matches_header():
    """ctypes g6r_frame mirrors include/g6r.h field for field (the host-copy
    pointers sit after the background colour)."""
    text = open(os.path.join(ROOT, "include", "g6r.h")).read()
    body = text[text.index("typedef struct g6r_frame {"):text.index("} g6r_frame;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\**\s*([a-z_0-9]+)(?:\[\d+\])?;", body)
    assert names == [f[0] for f in nat.Frame._fields_]
    assert ctypes.sizeof(nat.Frame) == 7 * 8 + 3 * 8 + 2 * 8


def test_workspace_size_grows_with_capacity():
    lib = nat.load()
    a = lib.g6r_workspace_bytes(1000, 64, 1 << 16, 0)
    b = lib.g6r_workspace_bytes(1000, 64, 1 << 20, 0)
    c = lib.g6r_workspace_bytes(1000, 64, 1 << 20, 1)
    assert 0 < a < b < c
    assert b - a >= ((1 << 20) - (1 << 16)) * 24   # keys+values, double-buffered


def test_abi_rejects_bad_arguments_before_touching_the_device():
    lib = nat.load()
    cam = nat.Camera()
    cam.width = cam.height = 64
    cam.focal = 70.0
    cfg = nat.Config(16, 0, 0.3, 0.99)
    sc = nat.Scene(10, None, None)
    fr = nat.Frame()
    rc = lib.g6r_render(ctypes.byref(sc), 0xFFFF, ctypes.byref(cam), ctypes.byref(cfg), None, 0, 0,
                        ctypes.byref(fr), None, None)
    assert rc == nat.G6R_EINVAL
    assert b"NULL" in lib.g6r_last_error()
    bad = nat.Config(64, 0, 0.3, 0.99)
    sc0 = nat.Scene(0, None, None)
    fr1 = nat.Frame(1, 1, 1, 1, 0, 0)
    rc = lib.g6r_render(ctypes.byref(sc0), 0xFFFF, ctypes.byref(cam), ctypes.byref(bad), None, 0, 0,
                        ctypes.byref(fr1), None, None)
    assert rc == nat.G6R_EINVAL and b"tile_size" in lib.g6r_last_error()
    rc = lib.g6r_render(ctypes.byref(sc0), 0xFFFF, ctypes.byref(cam), ctypes.byref(cfg), None, 0,
                        1 << 31, ctypes.byref(fr1), None, None)
    assert rc == nat.G6R_EINVAL and b"entry_capacity" in lib.g6r_last_error()
    rc = lib.g6r_render(ctypes.byref(sc0), 0xFFFF, ctypes.byref(cam), ctypes.byref(cfg), None, 0,
                        1024, ctypes.byref(fr1), None, None)
    assert rc == nat.G6R_EINVAL and b"workspace" in lib.g6r_last_error()
    bad_exp = nat.Config(16, 0, 0.3, 0.99, 2, 0)
    rc = lib.g6r_render(ctypes.byref(sc0), 0xFFFF, ctypes.byref(cam), ctypes.byref(bad_exp), None, 0,
                        0, ctypes.byref(fr1), None, None)
    assert rc == nat.G6R_EINVAL and b"exp_mode" in lib.g6r_last_error()


def test_exp_mode_is_validated_on_the_host():
    from paper_2505_17338_b200 import raster
    from paper_2505_17338_b200.errors import InvalidParameterError
    assert raster._check_config(raster.RenderConfig(exp_mode="fast")).exp_mode == 1
    assert raster._check_config(raster.RenderConfig()).exp_mode == 0
    with pytest.raises(InvalidParameterError):
        raster._check_config(raster.RenderConfig(exp_mode="approx"))


def test_check_maps_codes_to_exceptions():
    with pytest.raises(nat.G6RError) as ei:
        nat.check(nat.G6R_EINVAL)
    assert ei.value.code == nat.G6R_EINVAL


# --- config / masks / policy -----------------------------------------------

def test_render_config_validation():
    assert raster.RenderConfig().dtype() is np.float32
    assert raster.RenderConfig(precision="f64").dtype() is np.float64
    with pytest.raises(InvalidParameterError):
        raster.RenderConfig(precision="f16").dtype()
    with pytest.raises(InvalidParameterError):
        raster._check_config(raster.RenderConfig(tile_size=48))
    with pytest.raises(InvalidParameterError):
        raster._check_config(raster.RenderConfig(backend="opencl"))
    cfg = raster._check_config(raster.RenderConfig(precision="f64", tile_size=8))
    assert (cfg.tile_size, cfg.precision) == (8, 1)


def test_normalize_group_mask():
    m = raster.normalize_group_mask([2, 5, 7])
    assert m.dtype == bool and m.sum() == 3 and m[2] and m[5] and m[7]
    b = np.zeros(12, dtype=bool)
    b[[3, 4]] = True
    np.testing.assert_array_equal(raster.normalize_group_mask(b), b)
    with pytest.raises(InvalidParameterError):
        raster.normalize_group_mask([12])
    with pytest.raises(InvalidParameterError):
        raster.normalize_group_mask(np.zeros(5, dtype=bool))


class FakePrep:
    def __init__(self, labels, degenerate):
        labels = np.asarray(labels)
        self.n = len(labels)
        self.label_counts = np.zeros(32, dtype=np.int64)
        self.label_counts[:16] = np.bincount(labels, minlength=16)
        self.label_counts[16:] = np.bincount(labels[np.asarray(degenerate)], minlength=16)


def test_degenerate_policy_matches_reference_rule():
    # 3/300 degenerate is exactly the 1% limit: allowed; masking to their group: refused
    labels = np.concatenate([np.full(3, 9), np.full(297, 8)])
    deg = np.zeros(300, dtype=bool)
    deg[:3] = True
    prep = FakePrep(labels, deg)
    stats = raster.RenderStats()
    bits = raster._selection(prep, None, raster.DEFAULT_CONFIG, stats)
    assert bits == raster._ALL and stats.n_selected == 300 and stats.n_degenerate == 3
    with pytest.raises(DegenerateCovarianceError):
        raster._selection(prep, [9], raster.DEFAULT_CONFIG, raster.RenderStats())
    stats = raster.RenderStats()
    bits = raster._selection(prep, [8, 2], raster.DEFAULT_CONFIG, stats)
    assert bits == (1 << 8) | (1 << 2) and stats.n_selected == 297 and stats.n_degenerate == 0
    # 4 degenerate of 300 exceeds the limit
    deg[3] = True
    with pytest.raises(DegenerateCovarianceError):
        raster._selection(FakePrep(labels, deg), None, raster.DEFAULT_CONFIG, raster.RenderStats())


# --- input contracts --------------------------------------------------------

def test_camera_contract():
    cam = make_camera((0.0, 0.0, 70.0), (0.0, 0.0, 0.0), width=64, height=48)
    assert cam.focal == pytest.approx(48 / (2 * np.tan(0.4)))
    assert (cam.cx, cam.cy) == (31.5, 23.5)
    np.testing.assert_allclose(cam.rotation @ cam.rotation.T, np.eye(3), atol=1e-12)
    with pytest.raises(DegenerateGeometryError):
        make_camera((1.0, 2.0, 3.0), (1.0, 2.0, 3.0))
    with pytest.raises(InvalidParameterError):
        Camera(position=np.zeros(3), rotation=np.eye(3) * 2, fov_y=0.8, width=8, height=8)


def test_scene_contract_and_filter():
    s = scenes.random_scene(np.random.default_rng(0), 50)
    assert len(s) == 50 and s.labels.dtype == np.uint8
    f = filter_scene(s, [3, 4])
    assert np.all(np.isin(f.labels, [3, 4]))
    with pytest.raises(InvalidParameterError):
        Scene(mu_p=np.zeros((2, 3)), mu_d=np.zeros((2, 3)), cov_raw=np.zeros((2, 21)),
              sh=np.zeros((2, 12)), opacity_raw=np.zeros(2), labels=np.array([0, 1]))
    with pytest.raises(InvalidParameterError):
        Scene(mu_p=np.full((1, 3), np.nan), mu_d=np.zeros((1, 3)), cov_raw=np.zeros((1, 21)),
              sh=np.zeros((1, 12)), opacity_raw=np.zeros(1), labels=np.array([1]))


# --- scenes (benchmark workloads) -------------------------------------------

def digest(scene):
    h = hashlib.sha256()
    for f in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
        h.update(np.ascontiguousarray(getattr(scene, f)).tobytes())
    return h.hexdigest()[:16]


def test_scene_generators_match_reference(ref):
    from splatct import bench
    from splatct.phantom import make_phantom
    from splatct.priming import ParamVolume, decode_param_volume
    from splatct.volume import build_input_channels, consolidate_labels, load_preset, normalize_hu
    want = bench.benchmark_scene(2000, dims=(24, 24, 24))
    got = scenes.phantom_agp_scene((24, 24, 24)).take(np.arange(2000))
    assert digest(want) == digest(got)
    d = 40
    vol, labels = make_phantom((d,) * 3)
    g = consolidate_labels(labels)
    in6 = build_input_channels(normalize_hu(vol, labels), g, load_preset("seen"), vol)
    half = tuple(k // 2 for k in in6.dims)
    rng = np.random.default_rng(2505)
    ch = np.empty((37,) + half)
    ch[0:3] = rng.normal(0, 0.3, (3,) + half)
    ch[3:6] = rng.normal(0, 0.3, (3,) + half)
    ch[6:15] = rng.normal(0, 0.2, (9,) + half)
    ch[15] = rng.normal(0, 1.0, half)
    ch[16:22] = rng.uniform(-0.5, 0.3, (6,) + half)
    ch[22:37] = rng.normal(0, 0.3, (15,) + half)
    want = decode_param_volume(ParamVolume(channels=ch), in6, g)
    assert digest(want) == digest(scenes.psi_decode_scene(d))
    cw, cg = bench.benchmark_camera(want, 96, 80), scenes.benchmark_camera(want, 96, 80)
    np.testing.assert_array_equal(cw.position, cg.position)
    np.testing.assert_array_equal(cw.rotation, cg.rotation)


def test_scene_generators_are_deterministic():
    a = scenes.phantom_agp_scene((20, 20, 20))
    b = scenes.phantom_agp_scene((20, 20, 20))
    assert digest(a) == digest(b) and len(a) > 1000
    c = scenes.psi_decode_scene(32)
    assert len(c) > 500 and np.all(np.isfinite(c.cov_raw))
    ring = scenes.orbit_ring(c, count=8, size=64)
    assert len(ring) == 8 and ring[0].width == 64


# --- view sharding ------------------------------------------------------------

def test_shard_views_partition():
    for v in (1, 7, 100, 800):
        for w in (1, 2, 3, 4, 8):
            blocks = [multigpu.shard_views(v, w, r) for r in range(w)]
            flat = [i for b in blocks for i in b]
            assert flat == list(range(v))
            sizes = [len(b) for b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        multigpu.shard_views(10, 2, 2)


def test_pack_unpack_scene_roundtrip():
    import torch
    s = scenes.random_scene(np.random.default_rng(3), 33)
    ds = multigpu.unpack_scene(*multigpu.pack_scene(s, torch.device("cpu")))
    for f in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
        np.testing.assert_array_equal(getattr(ds, f).numpy(), getattr(s, f))
    np.testing.assert_array_equal(ds.spatial_scale, s.spatial_scale)
    assert len(ds) == 33


def test_scene_file_roundtrip_and_format_errors(tmp_path):
    from paper_2505_17338_b200 import sceneio
    s = scenes.random_scene(np.random.default_rng(4), 257)
    p = tmp_path / "a.g6ds"
    sceneio.save_scene(s, p)
    assert p.stat().st_size == 16 + 152 + 257 * 168
    t = sceneio.load_scene(p)
    for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw"):
        np.testing.assert_array_equal(getattr(t, k), getattr(s, k).astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(t.labels, s.labels)
    sceneio.save_scene(t, tmp_path / "b.g6ds")   # load-save-load is bit-stable
    assert (tmp_path / "b.g6ds").read_bytes() == p.read_bytes()
    blob = p.read_bytes()
    for bad, msg in ((b"XXXX" + blob[4:], "magic"), (blob[:4] + b"\x02" + blob[5:], "version"),
                     (blob[:-1], "payload"), (blob[:20], "short")):
        (tmp_path / "c.g6ds").write_bytes(bad)
        with pytest.raises(sceneio.SceneFormatError, match=msg):
            sceneio.load_scene(tmp_path / "c.g6ds")


def test_scene_file_bytes_match_reference_writer(ref, tmp_path):
    from splatct import sceneio as RS
    from splatct.priming import Scene as RScene
    from paper_2505_17338_b200 import sceneio
    s = scenes.random_scene(np.random.default_rng(8), 100)
    rs = RScene(mu_p=s.mu_p, mu_d=s.mu_d, cov_raw=s.cov_raw, sh=s.sh, opacity_raw=s.opacity_raw,
                labels=s.labels, spacing=np.array([1.5, 1.5, 2.0]), origin=np.array([1.0, 2, 3]),
                direction=np.eye(3)[[1, 0, 2]], spatial_scale=np.array([0.5, 1.0, 2.0]),
                directional_scale=0.7)
    RS.save_scene(rs, tmp_path / "r.g6ds")
    sceneio.save_scene(rs, tmp_path / "m.g6ds")
    assert (tmp_path / "r.g6ds").read_bytes() == (tmp_path / "m.g6ds").read_bytes()
    t = sceneio.load_scene(tmp_path / "r.g6ds")
    np.testing.assert_array_equal(t.direction, rs.direction)
    assert t.directional_scale == 0.7


def test_loss_config_and_polylr_match_reference_rules():
    from paper_2505_17338_b200 import diffrender as D
    c = D.LossConfig()
    assert abs(sum(c.ms_ssim_weights) - 1.0) < 1e-15
    for kw in (dict(lambda_l1=-1.0), dict(lambda_l1=0.0, lambda_ssim=0.0), dict(ms_ssim_scales=0),
               dict(ms_ssim_scales=2), dict(ms_ssim_weights=(1, 1, 1, 1, 0))):
        with pytest.raises(InvalidParameterError):
            D.LossConfig(**kw)
    assert D.polylr(0, 10, 1e-3) == 1e-3
    assert D.polylr(10, 10, 1e-3) == 0.0
    assert D.polylr(3, 10, 2e-3) == 2e-3 * (1.0 - 3 / 10) ** 0.9
    with pytest.raises(InvalidParameterError):
        D.polylr(11, 10, 1e-3)
    with pytest.raises(InvalidParameterError):
        D.finetune(scenes.random_scene(np.random.default_rng(0), 3), [])


def test_train_entry_points_reject_bad_arguments():
    import ctypes
    lib = nat.load()
    parts = (ctypes.c_double * 3)()
    w = (ctypes.c_double * 5)(*([0.2] * 5))
    # null pointers, bad channel count, tiny image, bad scales: rejected on the host
    assert lib.g6r_loss_grad(None, None, 3, 64, 64, 0.8, 0.2, 5, w, None, 0, None, parts,
                             None) == nat.G6R_EINVAL
    dummy = ctypes.c_void_p(256)
    assert lib.g6r_loss_grad(dummy, dummy, 2, 64, 64, 0.8, 0.2, 5, w, dummy, 1 << 30, dummy,
                             parts, None) == nat.G6R_EINVAL
    assert lib.g6r_loss_grad(dummy, dummy, 3, 8, 64, 0.8, 0.2, 5, w, dummy, 1 << 30, dummy,
                             parts, None) == nat.G6R_EINVAL
    assert lib.g6r_loss_grad(dummy, dummy, 3, 64, 64, 0.8, 0.2, 6, w, dummy, 1 << 30, dummy,
                             parts, None) == nat.G6R_EINVAL
    assert lib.g6r_loss_grad(dummy, dummy, 3, 64, 64, 0.8, 0.2, 5, w, dummy, 16, dummy,
                             parts, None) == nat.G6R_EINVAL
    assert lib.g6r_loss_workspace_bytes(64, 64) > 64 * 64 * 8 * 20
    assert lib.g6r_loss_workspace_bytes(0, 64) == 0
    assert lib.g6r_adam_step(-1, None, None, None, None, 1e-3, 0.1, 0.001, None) == nat.G6R_EINVAL
    assert lib.g6r_adam_step(0, None, None, None, None, 1e-3, 0.1, 0.001, None) == nat.G6R_OK
    assert lib.g6r_any_nonfinite(-1, None, None, None) == nat.G6R_EINVAL
    assert lib.g6r_decode_records(-1, None, None, None, None, None, None, None, None,
                                  None) == nat.G6R_EINVAL
    assert lib.g6r_decode_records(4, ctypes.c_void_p(257), dummy, dummy, dummy, dummy, dummy,
                                  dummy, dummy, None) == nat.G6R_EINVAL


def test_camera_array_matches_camera_structs():
    """render_views' column-filled camera array is byte for byte the
    g6r_camera structs _camera_struct builds one by one."""
    import ctypes
    from paper_2505_17338_b200 import raster, scenes
    from paper_2505_17338_b200 import _native as nat
    cams = [scenes.orbit_camera(azimuth=0.37 * k, elevation=0.1 * k - 0.2, width=96 + k, height=64,
                                fov_y=0.5 + 0.1 * k) for k in range(5)]
    a = raster._camera_array(cams)
    arr = (nat.Camera * len(cams)).from_buffer(a)
    assert ctypes.sizeof(nat.Camera) == a.dtype.itemsize
    for k, c in enumerate(cams):
        assert bytes(arr[k]) == bytes(raster._camera_struct(c)), k


def test_frame_array_layout_matches_g6r_frame():
    """render_views' numpy frame records have g6r_frame's size and field
    offsets (the ctypes mirror of g6r.h)."""
    import ctypes
    from paper_2505_17338_b200 import raster
    from paper_2505_17338_b200 import _native as nat
    dt = raster._FRAME_DTYPE
    assert dt.itemsize == ctypes.sizeof(nat.Frame)
    for name, _ in nat.Frame._fields_:
        assert dt.fields[name][1] == getattr(nat.Frame, name).offset, name
    assert raster._CAMERA_DTYPE.itemsize == ctypes.sizeof(nat.Camera)
    for name, _ in nat.Camera._fields_:
        assert raster._CAMERA_DTYPE.fields[name][1] == getattr(nat.Camera, name).offset, name
