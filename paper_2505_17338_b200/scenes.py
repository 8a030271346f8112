"""Synthetic workloads for the benchmark configurations (BASELINE.json configs).

There is no network for real CT data or Render-FM checkpoints, so the
benchmark scenes are synthesised exactly as the reference harness would
produce them, restated here in numpy (host-side data generation, not part of
the render path):

* ``random_scene``: random well-conditioned 6D Gaussians (the reference
  tests' ``make_scene``, test_raster.py:40-59) -- config 1.
* ``phantom_agp_scene``: nested-ellipsoid CT phantom (phantom.py:27-71) ->
  label consolidation (volume.py:50-64) -> "seen" transfer functions
  (volume.py:407-503, tf_presets/seen_tf.txt) -> anatomy-guided priming, one
  Gaussian per foreground voxel (priming.py:147-191) -- config 2.
* ``psi_decode_scene``: the same phantom with a seeded 37-channel parameter
  volume decoded into a scene (priming.py:194-285), the stand-in for the
  Render-FM network output -- configs 3-5 (SURVEY.md 8d recipe, seed 2505).

Every value is a pointwise function of its voxel, so only the voxels a
recipe actually reads are evaluated (the decode path touches the even-index
half grid only); tests/test_scenes.py checks bit-identity with the reference.
"""

from __future__ import annotations

import math

import numpy as np

from .camera import make_camera
from .scene import Scene

SH_C0 = 0.28209479177387814
ALPHA_FLOOR = 1e-4
DEFAULT_MU_D = np.array([0.0, 0.0, 1.0])

# phantom.py:19-33: (raw label, semi-axes as fractions of the half extent,
# boundary HU, HU rise to the centre), outermost first; raw labels 10/5/30
# consolidate to groups 5 (lung), 2 (liver), 7 (skeleton) (volume.py:50-64).
_REGIONS = ((5, (0.84, 0.72, 0.62), -850.0, 100.0),
            (2, (0.52, 0.44, 0.36), 120.0, 60.0),
            (7, (0.24, 0.18, 0.14), 700.0, 300.0))
_HU_AIR = -1000.0

# "seen" transfer-function ramps (tf_presets/seen_tf.txt) for the groups the
# phantom produces: rows of (HU, R, G, B, A) with colours in 0-255.
_SEEN_TF = {
    2: np.array([[-1024, 0, 0, 0, 0], [-20, 0, 0, 0, 0], [30, 100, 70, 50, 0.1],
                 [90, 140, 100, 70, 0.3], [180, 170, 130, 90, 0.6], [250, 190, 150, 110, 0.75],
                 [3072, 210, 170, 130, 0.85]], dtype=np.float64),
    5: np.array([[-1024, 0, 0, 0, 0], [-850, 190, 180, 180, 0.0008], [-500, 210, 200, 200, 0.0025],
                 [0, 230, 220, 220, 0.004], [1000, 240, 230, 230, 0.006],
                 [3072, 245, 235, 235, 0.008]], dtype=np.float64),
    7: np.array([[-1024, 0, 0, 0, 0], [100, 180, 30, 30, 0.1], [180, 255, 215, 140, 0.6],
                 [280, 255, 240, 240, 0.9], [350, 255, 255, 255, 1.0],
                 [3072, 255, 255, 255, 1.0]], dtype=np.float64),
}


def random_scene(rng, n, box=22.0, iso=False, opacity_lo=0.5, opacity_hi=3.0) -> Scene:
    """Random well-conditioned scene centred on the origin (config 1)."""
    mu_d = rng.normal(size=(n, 3))
    mu_d /= np.linalg.norm(mu_d, axis=1, keepdims=True)
    cov_raw = np.zeros((n, 21))
    if not iso:
        cov_raw[:, :6] = rng.uniform(-0.3, 0.8, size=(n, 6))
        cov_raw[:, 6:] = rng.normal(0.0, 0.35, size=(n, 15))
    return Scene(mu_p=rng.uniform(-box, box, size=(n, 3)), mu_d=mu_d, cov_raw=cov_raw,
                 sh=rng.normal(0.0, 0.4, size=(n, 12)),
                 opacity_raw=rng.uniform(opacity_lo, opacity_hi, size=n),
                 labels=rng.integers(1, 12, size=n), spacing=np.ones(3), origin=np.zeros(3),
                 direction=np.eye(3), spatial_scale=np.full(3, 3.0))


def _phantom(dims, spacing, step):
    """Raw-HU intensities and consolidated groups of the phantom on the voxel
    lattice ``[::step]`` along each axis (phantom.py:36-71)."""
    d, h, w = dims
    spacing = np.asarray(spacing, dtype=np.float64)
    nx = np.array([w, h, d], dtype=np.float64)
    half_extent = nx * spacing / 2.0
    origin = -(nx - 1) / 2.0 * spacing
    xs = origin[0] + np.arange(w) * spacing[0]
    ys = origin[1] + np.arange(h) * spacing[1]
    zs = origin[2] + np.arange(d) * spacing[2]
    x = xs[::step][None, None, :]
    y = ys[::step][None, :, None]
    z = zs[::step][:, None, None]
    shape = (len(zs[::step]), len(ys[::step]), len(xs[::step]))
    hu = np.full(shape, _HU_AIR)
    groups = np.zeros(shape, dtype=np.uint8)
    for group, fractions, hu_base, hu_rise in _REGIONS:
        ax, ay, az = np.asarray(fractions) * half_extent
        u = np.sqrt((x / ax) ** 2 + (y / ay) ** 2 + (z / az) ** 2)
        inside = u <= 1.0
        hu[inside] = hu_base + hu_rise * (1.0 - u[inside])
        groups[inside] = group
    return hu, groups, origin, spacing


def _tf_rgba(groups_fg, hu_fg):
    """Transfer-function RGBA (colours /255) per foreground voxel (volume.py:407-503)."""
    rgba = np.zeros((len(hu_fg), 4))
    for g, table in _SEEN_TF.items():
        sel = groups_fg == g
        if sel.any():
            out = np.stack([np.interp(hu_fg[sel], table[:, 0], table[:, 1 + c]) for c in range(4)],
                           axis=-1)
            out[:, :3] /= 255.0
            rgba[sel] = out
    return rgba


def phantom_agp_scene(dims=(128, 128, 128), spacing=(1.5, 1.5, 1.5), stride=1) -> Scene:
    """One Gaussian per foreground voxel primed from the TF colours (config 2)."""
    hu, groups, origin, spacing = _phantom(dims, spacing, stride)
    zi, yi, xi = np.nonzero(groups)
    index_xyz = np.stack([xi, yi, zi], axis=1) * stride
    mu_p = origin + (index_xyz * spacing) @ np.eye(3).T
    rgba = _tf_rgba(groups[zi, yi, xi], hu[zi, yi, xi])
    alpha = np.clip(rgba[:, 3], ALPHA_FLOOR, 1.0 - ALPHA_FLOOR)
    n = zi.size
    sh = np.zeros((n, 12))
    sh[:, :3] = (rgba[:, :3] - 0.5) / SH_C0
    return Scene(mu_p=mu_p, mu_d=np.tile(DEFAULT_MU_D, (n, 1)), cov_raw=np.zeros((n, 21)), sh=sh,
                 opacity_raw=np.log(alpha / (1.0 - alpha)), labels=groups[zi, yi, xi],
                 spacing=spacing, origin=origin, direction=np.eye(3),
                 spatial_scale=spacing * stride / 2.0, directional_scale=1.0)


def psi_decode_scene(dim=352, seed=2505, spacing=(1.5, 1.5, 1.5), limit=None) -> Scene:
    """Decode a seeded 37-channel parameter volume on the phantom's half grid
    (configs 3-5: dim 352 gives 1,070,404 Gaussians; take the first 1M)."""
    dims = (dim, dim, dim)
    half = tuple(d // 2 for d in dims)
    hu, groups, origin, spacing = _phantom(dims, spacing, 2)
    hu, groups = hu[:half[0], :half[1], :half[2]], groups[:half[0], :half[1], :half[2]]
    zi, yi, xi = np.nonzero(groups)
    rng = np.random.default_rng(seed)
    # channel draws in the recipe's order, each gathered at the foreground
    draws = [(3, "normal", 0.3), (3, "normal", 0.3), (9, "normal", 0.2), (1, "normal", 1.0),
             (6, "uniform", None), (15, "normal", 0.3)]
    pred = []
    for k, kind, s in draws:
        shape = (k,) + half if k > 1 else half
        block = rng.normal(0, s, shape) if kind == "normal" else rng.uniform(-0.5, 0.3, shape)
        block = block.reshape((k,) + half)
        pred.append(block[:, zi, yi, xi])
        del block
    pred = np.concatenate(pred, axis=0)
    n = zi.size
    index_xyz = np.stack([xi, yi, zi], axis=1) * 2
    mu_p = origin + (index_xyz * spacing) @ np.eye(3).T
    rgba = _tf_rgba(groups[zi, yi, xi], hu[zi, yi, xi])
    sh = np.zeros((n, 12))
    sh[:, :3] = (rgba[:, :3] - 0.5) / SH_C0 + pred[3:6].T
    sh[:, 3:] = pred[6:15].T
    cov_raw = np.empty((n, 21))
    cov_raw[:, :6] = pred[16:22].T
    cov_raw[:, 6:] = pred[22:37].T
    scene = Scene(mu_p=mu_p, mu_d=DEFAULT_MU_D + pred[0:3].T, cov_raw=cov_raw, sh=sh,
                  opacity_raw=rgba[:, 3] + pred[15], labels=groups[zi, yi, xi], spacing=spacing,
                  origin=origin, direction=np.eye(3), spatial_scale=spacing,
                  directional_scale=1.0)
    if limit is not None:
        scene = scene.take(np.arange(min(limit, len(scene))))
    return scene


def benchmark_camera(scene, width=512, height=512):
    """Camera framing the whole scene from a fixed oblique direction (bench.py:57-66)."""
    lo = scene.mu_p.min(axis=0)
    hi = scene.mu_p.max(axis=0)
    center = (lo + hi) / 2.0
    radius = float(np.linalg.norm(hi - lo)) / 2.0
    fov_y = 0.8
    distance = 1.2 * radius / np.tan(fov_y / 2.0)
    position = center + distance * np.array([0.45, 0.35, 0.82])
    return make_camera(position, center, fov_y=fov_y, width=width, height=height)


def orbit_ring(scene, count=100, size=512, fov=0.8):
    """Ring of cameras around the scene's bounding box at two elevations
    (test_acceptance.py:131-146, the orbit of configs 3-4)."""
    lo = scene.mu_p.min(axis=0)
    hi = scene.mu_p.max(axis=0)
    center = (lo + hi) / 2.0
    radius = float(np.linalg.norm(hi - lo)) / 2.0
    distance = 1.2 * radius / np.tan(fov / 2.0)
    cams = []
    for k in range(count):
        az = 2.0 * np.pi * k / count
        el = 0.35 if k % 2 else -0.2
        offset = np.array([np.cos(el) * np.sin(az), np.sin(el), np.cos(el) * np.cos(az)])
        cams.append(make_camera(center + distance * offset, center, fov_y=fov, width=size,
                                height=size))
    return cams


def orbit_camera(azimuth=0.0, elevation=0.0, distance=70.0, width=64, height=64, fov_y=0.8,
                 target=(0.0, 0.0, 0.0)):
    """Single orbit camera about ``target`` (test_raster.py:62-70)."""
    target = np.asarray(target, dtype=np.float64)
    ce, se = math.cos(elevation), math.sin(elevation)
    ca, sa = math.cos(azimuth), math.sin(azimuth)
    position = target + distance * np.array([sa * ce, se, ca * ce])
    return make_camera(position, target, fov_y=fov_y, width=width, height=height)


def synthetic_target(width, height, seed=0, channels=4) -> np.ndarray:
    """A smooth (H, W, channels) f64 target image for fine-tune runs and tests.

    Polynomial in the pixel coordinates with seeded coefficients: only +, -, *
    so it regenerates bit for bit on any host (no transcendental ufuncs)."""
    c = np.random.default_rng(seed).uniform(0.05, 0.45, (3, 4))
    u = (np.arange(width, dtype=np.float64) + 0.5) / width
    v = (np.arange(height, dtype=np.float64) + 0.5) / height
    u, v = np.meshgrid(u, v)
    img = np.ones((height, width, channels))
    for k in range(3):
        img[:, :, k] = c[k, 0] + c[k, 1] * u + c[k, 2] * v * v + c[k, 3] * u * v * (1.0 - u)
    return img
