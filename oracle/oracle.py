"""CPU oracle for the 6DGS render path -- TEST INFRASTRUCTURE ONLY.

Restates the reference renderer (splatct 0.1.0, ``/root/reference/pkg/src/splatct``)
as a checker for the CUDA path: numpy for the per-scene preparation and the
binning/sort (so transcendentals come from the same numpy ufuncs the reference
calls), and the C restatement in ``g6r_oracle.c`` for the per-Gaussian
projection and per-pixel compositing loops.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg
may import this module.  The product package never does.

Parity is pinned two ways (tests/test_oracle.py): bit-identity with the compiled
reference itself (``oracle/_ref``, built by ``oracle/build_ref.sh``) and with the
golden fixtures committed under ``tests/golden`` (made by
``tests/golden/make_golden.py`` from the reference).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libg6r_oracle.so")

# Reference constants: core.py:25-26 (SH), raster.py:47 (MIN_ALPHA),
# core.py:30-31 (row-major strict-lower index pairs of the 6x6 factor).
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
MIN_ALPHA = 1.0 / 255.0
TRIL_I = np.array([1, 2, 2, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 5])
TRIL_J = np.array([0, 1, 0, 0, 1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 4])
N_GROUPS = 12


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile g6r_oracle.c into oracle/build (gcc, -ffp-contract=off)."""
    src = os.path.join(HERE, "g6r_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.or_project_stage1.argtypes = [I64, P, P, P, P, D, D, D, P, P, P, P]
        L.or_project_stage2.argtypes = [I64, P, P, P, P, P, D, D, D, D, D, D, D, D, D, D,
                                        D, D, D, D, D, P, P, P, P, P, P]
        for name in ("or_composite_f32", "or_composite_f64"):
            getattr(L, name).argtypes = [P, P, P, P, P, P, I64, I, I, I, I, P, P, P]
        L.or_composite_backward.argtypes = [P, P, P, P, P, P, I64, I, I, I, I, P, P, P, P]
        L.or_expf_glibc_batch.argtypes = [I64, P, P]
        L.or_libm_exp_batch.argtypes = [I64, P, P]
        L.or_fma_batch.argtypes = [I64, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# Per-scene preparation (view-independent terms).  core.py:54-62, 255-351.
# ---------------------------------------------------------------------------

def sigmoid(x):
    """Stable logistic, same branch split as core.py:54-62."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def cholesky_factor(cov_raw, spatial_scale, directional_scale):
    """(N,21) raws -> (N,6,6) lower factors.  core.py:255-266."""
    raw = np.asarray(cov_raw, dtype=np.float64)
    n = raw.shape[0]
    scale = np.empty(6)
    scale[:3] = spatial_scale
    scale[3:] = directional_scale
    L = np.zeros((n, 6, 6))
    d = np.arange(6)
    L[:, d, d] = scale * np.exp(raw[:, :6])
    L[:, TRIL_I, TRIL_J] = np.tanh(raw[:, 6:])
    return L


def covariance(L):
    """Sigma = L L^T with numpy einsum's summation order for this contraction
    (core.py:269-272): ((p0+p2)+p4) + ((p1+p3)+p5), p_j = L[i,j] L[k,j]."""
    p = L[:, :, None, :] * L[:, None, :, :]          # (N,6,6,6): p[n,i,k,j]
    return ((p[..., 0] + p[..., 2]) + p[..., 4]) + ((p[..., 1] + p[..., 3]) + p[..., 5])


def inv3(m):
    """Adjugate inverse and determinant of (N,3,3).  core.py:275-302."""
    a, b, c = m[:, 0, 0], m[:, 0, 1], m[:, 0, 2]
    d, e, f = m[:, 1, 0], m[:, 1, 1], m[:, 1, 2]
    g, h, i = m[:, 2, 0], m[:, 2, 1], m[:, 2, 2]
    co00 = e * i - f * h
    co01 = f * g - d * i
    co02 = d * h - e * g
    det = a * co00 + b * co01 + c * co02
    inv = np.empty_like(m)
    inv[:, 0, 0] = co00
    inv[:, 0, 1] = c * h - b * i
    inv[:, 0, 2] = b * f - c * e
    inv[:, 1, 0] = co01
    inv[:, 1, 1] = a * i - c * g
    inv[:, 1, 2] = c * d - a * f
    inv[:, 2, 0] = co02
    inv[:, 2, 1] = b * g - a * h
    inv[:, 2, 2] = a * e - b * d
    with np.errstate(divide="ignore", invalid="ignore"):
        inv /= det[:, None, None]
    return inv, det


@dataclass
class Prep:
    sigma: np.ndarray
    adjust: np.ndarray
    precision_dd: np.ndarray
    sigma_prime: np.ndarray
    w_norm: np.ndarray
    degenerate: np.ndarray
    opacity: np.ndarray


def prepare(scene, w_mode: str = "peak", chunk: int = 65536) -> Prep:
    """View-independent slicing terms.  raster.py:120-137, core.py:324-351.
    Row-elementwise, so chunking over rows does not change any bit."""
    n = len(scene.mu_p)
    if n > chunk:
        parts = [_prepare_rows(scene.cov_raw[i:i + chunk], scene.opacity_raw[i:i + chunk],
                               scene.spatial_scale, scene.directional_scale, w_mode)
                 for i in range(0, n, chunk)]
        return Prep(*[np.concatenate([getattr(p, f) for p in parts])
                      for f in ("sigma", "adjust", "precision_dd", "sigma_prime",
                                "w_norm", "degenerate", "opacity")])
    return _prepare_rows(scene.cov_raw, scene.opacity_raw, scene.spatial_scale,
                         scene.directional_scale, w_mode)


def _prepare_rows(cov_raw, opacity_raw, spatial_scale, directional_scale, w_mode):
    L = cholesky_factor(cov_raw, spatial_scale, directional_scale)
    S = covariance(L)
    pp, pd, dd = S[:, :3, :3], S[:, :3, 3:], S[:, 3:, 3:]
    P, det = inv3(dd)
    trace = (dd[:, 0, 0] + dd[:, 1, 1]) + dd[:, 2, 2]
    with np.errstate(invalid="ignore", over="ignore"):
        degenerate = ~np.isfinite(det) | (det <= 1e-30 * np.maximum(trace, 1e-30) ** 3)
    P[degenerate] = 0.0
    # adjust[i,k] = (pd[i,0]P[0,k] + pd[i,1]P[1,k]) + pd[i,2]P[2,k]
    adj = (pd[:, :, 0, None] * P[:, None, 0, :] + pd[:, :, 1, None] * P[:, None, 1, :]) \
        + pd[:, :, 2, None] * P[:, None, 2, :]
    # sigma_prime[i,k] = pp[i,k] - ((q0 + q2) + q1), q_j = adj[i,j] pd[k,j]
    q = adj[:, :, None, :] * pd[:, None, :, :]
    sp = pp - ((q[..., 0] + q[..., 2]) + q[..., 1])
    if w_mode == "peak":
        w_norm = np.ones(S.shape[0])
    elif w_mode == "raw":
        with np.errstate(invalid="ignore", divide="ignore"):
            w_norm = (2.0 * np.pi) ** -1.5 / np.sqrt(det)
        w_norm[degenerate] = 0.0
    else:
        raise ValueError(f"unknown opacity modulation mode {w_mode!r}")
    return Prep(sigma=S, adjust=adj, precision_dd=P, sigma_prime=sp, w_norm=w_norm,
                degenerate=degenerate, opacity=sigmoid(opacity_raw))


def group_mask_bool(group_mask):
    """raster.py:140-154 without the error types (oracle input is trusted)."""
    arr = np.asarray(group_mask)
    if arr.dtype == bool:
        return arr.copy()
    mask = np.zeros(N_GROUPS, dtype=bool)
    for g in np.atleast_1d(arr):
        mask[int(g)] = True
    return mask


def select_rows(scene, prep: Prep, group_mask, degenerate_limit=0.01):
    """raster.py:418-440.  Returns (rows, n_selected, n_degenerate); raises
    OracleError where the reference raises DegenerateCovarianceError."""
    if group_mask is None:
        selected = np.arange(len(scene.mu_p), dtype=np.int64)
    else:
        selected = np.nonzero(group_mask_bool(group_mask)[scene.labels])[0]
    deg = prep.degenerate[selected]
    n_bad = int(deg.sum())
    if selected.size and n_bad > degenerate_limit * selected.size:
        raise OracleError("degenerate")
    return selected[~deg], int(selected.size), n_bad


# ---------------------------------------------------------------------------
# Projection.  raster.py:229-309 driving the C stage kernels.
# ---------------------------------------------------------------------------

@dataclass
class Splats:
    gids: np.ndarray
    means2d: np.ndarray
    conics: np.ndarray
    colors: np.ndarray
    alphas: np.ndarray
    depths: np.ndarray
    radii: np.ndarray
    stage: np.ndarray = field(repr=False, default=None)   # per selected row


def project(scene, prep: Prep, rows, camera, low_pass=0.3, alpha_max=0.99) -> Splats:
    L = lib()
    rows = np.asarray(rows, dtype=np.int64)
    mu_p = _c(scene.mu_p[rows], np.float64)
    mu_d = _c(scene.mu_d[rows], np.float64)
    adj = _c(prep.adjust[rows], np.float64)
    prec = _c(prep.precision_dd[rows], np.float64)
    n = len(rows)
    pos = np.asarray(camera.position, dtype=np.float64)
    px, py, pz = float(pos[0]), float(pos[1]), float(pos[2])
    stage = np.zeros(n, dtype=np.uint8)
    view = np.zeros((n, 3))
    mean_adj = np.zeros((n, 3))
    quad = np.zeros(n)
    L.or_project_stage1(n, _p(mu_p), _p(mu_d), _p(adj), _p(prec), px, py, pz,
                        _p(view), _p(mean_adj), _p(quad), _p(stage))
    # opacity modulation in numpy, as raster.py:258-261 does
    w = np.exp(-0.5 * quad) * prep.w_norm[rows]
    alphas = np.minimum(prep.opacity[rows] * w, alpha_max)
    stage[(stage == 0) & ~(alphas >= MIN_ALPHA)] = 2
    f = camera.height / (2.0 * np.tan(camera.fov_y / 2.0)) if not hasattr(camera, "focal") else camera.focal
    lim_x = 1.3 * camera.width / (2.0 * f)
    lim_y = 1.3 * camera.height / (2.0 * f)
    means2d = np.zeros((n, 2))
    conics = np.zeros((n, 3))
    colors = np.zeros((n, 3))
    depths = np.zeros(n)
    radii = np.zeros((n, 2), dtype=np.int32)
    sh = _c(scene.sh[rows], np.float64)
    sp = _c(prep.sigma_prime[rows], np.float64)
    rot = _c(camera.rotation, np.float64)
    cx = (camera.width - 1) / 2.0
    cy = (camera.height - 1) / 2.0
    L.or_project_stage2(n, _p(view), _p(mean_adj), _p(sh), _p(sp), _p(rot), px, py, pz,
                        float(camera.near), float(camera.far), f, cx, cy, lim_x, lim_y,
                        float(camera.width), float(camera.height), low_pass, SH_C0, SH_C1,
                        _p(means2d), _p(conics), _p(colors), _p(depths), _p(radii), _p(stage))
    kept = np.nonzero(stage == 0)[0]
    return Splats(gids=rows[kept], means2d=means2d[kept], conics=conics[kept],
                  colors=colors[kept], alphas=alphas[kept], depths=depths[kept],
                  radii=radii[kept], stage=stage)


# ---------------------------------------------------------------------------
# Binning.  raster.py:340-381.
# ---------------------------------------------------------------------------

@dataclass
class Entries:
    keys: np.ndarray          # sorted (tile << 32) | f32 depth bits
    entry_splat: np.ndarray   # int32
    tile_starts: np.ndarray   # int64 (T+1)
    tiles_x: int
    tiles_y: int


def bin_splats(means2d, radii, depths, width, height, tile_size=16) -> Entries:
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    n_tiles = tiles_x * tiles_y
    m = len(depths)
    if m == 0:
        return Entries(np.zeros(0, np.uint64), np.zeros(0, np.int32),
                       np.zeros(n_tiles + 1, np.int64), tiles_x, tiles_y)
    u, v = means2d[:, 0], means2d[:, 1]
    rx, ry = radii[:, 0], radii[:, 1]
    x0 = np.clip(np.floor((u - rx) / tile_size).astype(np.int64), 0, tiles_x - 1)
    x1 = np.clip(np.floor((u + rx) / tile_size).astype(np.int64), 0, tiles_x - 1)
    y0 = np.clip(np.floor((v - ry) / tile_size).astype(np.int64), 0, tiles_y - 1)
    y1 = np.clip(np.floor((v + ry) / tile_size).astype(np.int64), 0, tiles_y - 1)
    wx = x1 - x0 + 1
    counts = wx * (y1 - y0 + 1)
    start = np.concatenate([[0], np.cumsum(counts)])
    owner = np.repeat(np.arange(m, dtype=np.int64), counts)
    local = np.arange(start[-1], dtype=np.int64) - start[owner]
    tile = (y0[owner] + local // wx[owner]) * tiles_x + (x0[owner] + local % wx[owner])
    dbits = np.asarray(depths, np.float64).astype(np.float32).view(np.uint32).astype(np.uint64)
    key = (tile.astype(np.uint64) << np.uint64(32)) | dbits[owner]
    order = np.argsort(key, kind="stable")
    tile_starts = np.zeros(n_tiles + 1, dtype=np.int64)
    np.cumsum(np.bincount(tile, minlength=n_tiles), out=tile_starts[1:])
    return Entries(key[order], owner[order].astype(np.int32), tile_starts, tiles_x, tiles_y)


# ---------------------------------------------------------------------------
# Compositing.  raster.py:392-415.
# ---------------------------------------------------------------------------

def composite(means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
              tile_size, width, height, precision="f32"):
    dt = np.float32 if precision == "f32" else np.float64
    image = np.zeros((height, width, 4), dtype=dt)
    final_t = np.ones((height, width), dtype=dt)
    last = np.zeros((height, width), dtype=np.int32)
    args = [_c(means2d, dt), _c(conics, dt), _c(colors, dt), _c(alphas, dt),
            _c(entry_splat, np.int32), _c(tile_starts, np.int64)]
    fn = lib().or_composite_f32 if dt is np.float32 else lib().or_composite_f64
    fn(*[_p(a) for a in args], len(tile_starts) - 1, tiles_x, tile_size, width, height,
       _p(image), _p(final_t), _p(last))
    return image, final_t, last


def composite_backward(means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
                       tile_size, width, height, final_t, last_contrib, grad_image, init=0.0):
    """Per-entry gradient rows accumulated (+=) into rows filled with `init`."""
    e = len(entry_splat)
    grads = np.full((e, 9), float(init))
    args = [_c(means2d, np.float64), _c(conics, np.float64), _c(colors, np.float64),
            _c(alphas, np.float64), _c(entry_splat, np.int32), _c(tile_starts, np.int64)]
    tail = [_c(final_t, np.float64), _c(last_contrib, np.int32), _c(grad_image, np.float64)]
    lib().or_composite_backward(*[_p(a) for a in args], len(tile_starts) - 1, tiles_x,
                                tile_size, width, height, *[_p(a) for a in tail], _p(grads))
    return grads


@dataclass
class State:
    image: np.ndarray
    final_t: np.ndarray
    last_contrib: np.ndarray
    splats: Splats
    entries: Entries
    n_selected: int
    n_degenerate: int
    fate: np.ndarray        # bincount of stage codes over the projected rows


def render_with_state(scene, camera, group_mask=None, precision="f32", w_mode="peak",
                      tile_size=16, low_pass=0.3, alpha_max=0.99, prep: Prep | None = None) -> State:
    """raster.py:443-455 end to end."""
    prep = prep if prep is not None else prepare(scene, w_mode)
    rows, n_sel, n_bad = select_rows(scene, prep, group_mask)
    sp = project(scene, prep, rows, camera, low_pass, alpha_max)
    en = bin_splats(sp.means2d, sp.radii, sp.depths, camera.width, camera.height, tile_size)
    img, ft, last = composite(sp.means2d, sp.conics, sp.colors, sp.alphas, en.entry_splat,
                              en.tile_starts, en.tiles_x, tile_size, camera.width,
                              camera.height, precision)
    fate = np.bincount(sp.stage, minlength=6)
    return State(img, ft, last, sp, en, n_sel, n_bad, fate)


def render(scene, camera, group_mask=None, precision="f32", **kw):
    return render_with_state(scene, camera, group_mask, precision, **kw).image


def libm_exp(x):
    """The host libm exp (glibc 2.39) over a float64 array."""
    x = _c(x, np.float64)
    y = np.empty_like(x)
    lib().or_libm_exp_batch(x.size, _p(x), _p(y))
    return y


def expf_glibc(x):
    """glibc 2.39 expf model (g6r_oracle.c:or_expf_glibc) over a float32 array."""
    x = _c(x, np.float32)
    y = np.empty_like(x)
    lib().or_expf_glibc_batch(x.size, _p(x), _p(y))
    return y


def psnr(a, b):
    """PSNR over RGB in [0,1] (metrics.py:35-47 formula)."""
    d = np.asarray(a, np.float64)[..., :3] - np.asarray(b, np.float64)[..., :3]
    mse = float(np.mean(d * d))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)


# ---------------------------------------------------------------------------
# Photometric loss of the fine-tune loop (diffrender.py:117-138) and the
# multi-scale SSIM it uses (_ssim.py:23-201), restated with shifted-slice
# accumulation instead of sliding-window einsums.
# ---------------------------------------------------------------------------

_SSIM_C1 = 0.01 ** 2
_SSIM_C2 = 0.03 ** 2


def ssim_window(size=11, sigma=1.5):
    """_ssim.py:23-30: normalised 1-D Gaussian, centre (size-1)/2."""
    x = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-(x ** 2) / (2.0 * sigma ** 2))
    return g / g.sum()


def _corr(img, w, full=False):
    """Separable 2-D correlation, valid (or full = the adjoint) (_ssim.py:33-51)."""
    k = len(w)
    if full:
        img = np.pad(img, k - 1)
    h = img.shape[0] - k + 1
    t = sum(w[i] * img[i:i + h] for i in range(k))
    wv = img.shape[1] - k + 1
    return sum(w[i] * t[:, i:i + wv] for i in range(k))


def _pool(img):
    h2, w2 = img.shape[0] // 2, img.shape[1] // 2
    v = img[:2 * h2, :2 * w2]
    return 0.25 * (v[0::2, 0::2] + v[1::2, 0::2] + v[0::2, 1::2] + v[1::2, 1::2])


def _pool_adjoint(g, shape):
    out = np.zeros(shape)
    h2, w2 = g.shape
    out[:2 * h2, :2 * w2] = 0.25 * np.repeat(np.repeat(g, 2, axis=0), 2, axis=1)
    return out


def _ssim_level(x, y, w):
    ux, uy = _corr(x, w), _corr(y, w)
    sxx = _corr(x * x, w) - ux * ux
    syy = _corr(y * y, w) - uy * uy
    sxy = _corr(x * y, w) - ux * uy
    b1 = ux * ux + uy * uy + _SSIM_C1
    b2 = sxx + syy + _SSIM_C2
    return dict(x=x, y=y, ux=ux, uy=uy, b1=b1, b2=b2, l=(2.0 * ux * uy + _SSIM_C1) / b1,
                cs=(2.0 * sxy + _SSIM_C2) / b2)


def _ssim_level_backward(p, g_lcs, g_cs, w):
    """_ssim.py:86-98 with scalar per-window upstream gradients."""
    g_l = g_lcs * p["cs"]
    g_t = g_lcs * p["l"] + g_cs
    g_ux = (g_l * 2.0 * (p["uy"] - p["l"] * p["ux"]) / p["b1"]
            + g_t * 2.0 * (p["cs"] * p["ux"] - p["uy"]) / p["b2"])
    g_exx = -g_t * p["cs"] / p["b2"]
    g_exy = g_t * 2.0 / p["b2"]
    return (_corr(g_ux, w, True) + 2.0 * p["x"] * _corr(g_exx, w, True)
            + p["y"] * _corr(g_exy, w, True))


def ms_ssim_with_grad(a, b, scales=5, weights=(0.0448, 0.2856, 0.3001, 0.2363, 0.1333)):
    """Value and d/da of MS-SSIM over the channels of (H,W,C) images (_ssim.py:123-201)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    w = ssim_window()
    ns = 1 if min(a.shape[:2]) < (2 ** (scales - 1)) * 11 else scales
    wt = np.asarray(weights[:ns], np.float64)
    wt = wt / wt.sum()
    total, grad = 0.0, np.zeros(a.shape)
    for c in range(a.shape[2]):
        x, y, lv = a[:, :, c], b[:, :, c], []
        for j in range(ns):
            lv.append(_ssim_level(x, y, w))
            if j + 1 < ns:
                x, y = _pool(x), _pool(y)
        if ns == 1:
            p = lv[0]
            value = float(np.mean(p["l"] * p["cs"]))
            g = _ssim_level_backward(p, 1.0 / p["cs"].size, 0.0, w)
        else:
            terms = [max(float(np.mean(p["l"] * p["cs"])) if j == ns - 1 else
                         float(np.mean(p["cs"])), 0.0) for j, p in enumerate(lv)]
            value = float(np.prod(np.power(terms, wt)))
            g = np.zeros(lv[-1]["x"].shape)
            for j in range(ns - 1, -1, -1):
                p = lv[j]
                if j < ns - 1:
                    g = _pool_adjoint(g, p["x"].shape)
                if value > 0.0 and terms[j] > 0.0:
                    per = value * wt[j] / terms[j] / p["cs"].size
                    g = g + (_ssim_level_backward(p, per, 0.0, w) if j == ns - 1
                             else _ssim_level_backward(p, 0.0, per, w))
        total += value
        grad[:, :, c] = g
    n = a.shape[2]
    return total / n, grad / n


def loss_parts(pred, gt, lambda_l1=0.8, lambda_ssim=0.2, scales=5,
               weights=(0.0448, 0.2856, 0.3001, 0.2363, 0.1333)):
    """(total, l1, ssim_loss, d total / d pred) over RGB (diffrender.py:117-138)."""
    pred = np.asarray(pred, np.float64)
    p, g = pred[:, :, :3], np.asarray(gt, np.float64)[:, :, :3]
    d = p - g
    l1 = float(np.mean(np.abs(d)))
    grad = np.zeros(pred.shape)
    grad_rgb = lambda_l1 * np.sign(d) / d.size
    ssim_loss = 0.0
    if lambda_ssim > 0.0:
        wts = np.asarray(weights, np.float64)
        value, gm = ms_ssim_with_grad(p, g, scales, wts / wts.sum())
        ssim_loss = 1.0 - value
        grad_rgb = grad_rgb - lambda_ssim * gm
    grad[:, :, :3] = grad_rgb
    return lambda_l1 * l1 + lambda_ssim * ssim_loss, l1, ssim_loss, grad


# ---------------------------------------------------------------------------
# Scene ingest: Psi decode (priming.py:232-285), restated
# ---------------------------------------------------------------------------

def fma(a, b, c):
    """Correctly rounded a*b + c, broadcast (C99 fma via g6r_oracle.c)."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float64), np.asarray(b, np.float64),
                                  np.asarray(c, np.float64))
    a, b, c = (np.ascontiguousarray(x) for x in (a, b, c))
    out = np.empty_like(a)
    lib().or_fma_batch(a.size, _p(a), _p(b), _p(c), _p(out))
    return out


def decode_param_volume(psi, in6_channels, labels, spacing, origin, direction):
    """Scene rows (dict of arrays) for the foreground of the half grid.  World
    coordinates as origin + fma(q2, d[k,2], fma(q1, d[k,1], q0*d[k,0])) with
    q = index*2*spacing: the accumulation OpenBLAS dgemm performs for the
    reference's ``(index * spacing) @ direction.T`` (priming.py:134) on the
    reference host, pinned by tests/golden/ingest_rotated.npz."""
    psi = np.asarray(psi, np.float64)
    dp, hp, wp = psi.shape[1:]
    lab = np.asarray(labels)[::2, ::2, ::2][:dp, :hp, :wp]
    base = np.asarray(in6_channels, np.float64)[:, ::2, ::2, ::2][:, :dp, :hp, :wp]
    zi, yi, xi = np.nonzero(lab)
    q = np.stack([xi * 2, yi * 2, zi * 2], axis=1).astype(np.float64) * np.asarray(spacing, np.float64)
    d = np.asarray(direction, np.float64)
    mu_p = np.asarray(origin, np.float64) + fma(q[:, 2:3], d[:, 2], fma(q[:, 1:2], d[:, 1],
                                                                       q[:, 0:1] * d[:, 0]))
    pred = psi[:, zi, yi, xi]
    sh = np.empty((zi.size, 12))
    sh[:, :3] = (base[2:5, zi, yi, xi].T - 0.5) / SH_C0 + pred[3:6].T
    sh[:, 3:] = pred[6:15].T
    return dict(mu_p=mu_p, mu_d=np.array([0.0, 0.0, 1.0]) + pred[0:3].T,
                cov_raw=np.ascontiguousarray(pred[16:37].T), sh=sh,
                opacity_raw=base[5, zi, yi, xi] + pred[15], labels=lab[zi, yi, xi])
