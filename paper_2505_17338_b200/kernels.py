"""Kernel-module adapter with the reference backend contract.

The reference picks a kernel module by name (raster.py:50-82) exposing
``BACKEND``, ``project_stage1``, ``project_stage2``, ``composite_forward`` and
``composite_backward`` with host numpy arrays written in place
(_kernels.pyx:36-363).  This module has the same names and signatures; each
call uploads its inputs, runs the CUDA kernel behind the C ABI, and writes the
results back into the caller's arrays.  It lets the reference's kernel-level
tests (tests/test_raster.py:303-411 of the reference) be pointed at the B200
path; the product render path does not go through it.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .raster import _ptr, _require_cuda, _stream_handle, composite_arrays

BACKEND = "cuda"


def _dev():
    import torch
    _require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _up(a, dt):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(_dev())


def _down(t, out):
    out[...] = t.cpu().numpy().reshape(out.shape)


def project_stage1(mu_p, mu_d, adjust, precision_dd, px, py, pz, view, mean_adj, quad, stage,
                   threads=1):
    n = len(mu_p)
    ins = [_up(mu_p, np.float64), _up(mu_d, np.float64), _up(adjust, np.float64),
           _up(precision_dd, np.float64)]
    outs = [_up(view, np.float64), _up(mean_adj, np.float64), _up(quad, np.float64),
            _up(stage, np.uint8)]
    nat.check(nat.load().g6r_project_stage1(n, *[_ptr(t) for t in ins], float(px), float(py),
                                            float(pz), *[_ptr(t) for t in outs], _stream_handle()))
    for t, o in zip(outs, (view, mean_adj, quad, stage)):
        _down(t, o)


def project_stage2(view, mean_adj, sh, sigma_prime, rot, px, py, pz, near, far, f, ox, oy, lim_x,
                   lim_y, width, height, low_pass, sh_c0, sh_c1, means2d, conics, colors, depths,
                   radii, stage, threads=1):
    n = len(view)
    ins = [_up(view, np.float64), _up(mean_adj, np.float64), _up(sh, np.float64),
           _up(sigma_prime, np.float64)]
    rot9 = (ctypes.c_double * 9)(*np.asarray(rot, dtype=np.float64).reshape(9).tolist())
    outs = [_up(means2d, np.float64), _up(conics, np.float64), _up(colors, np.float64),
            _up(depths, np.float64), _up(radii, np.int32), _up(stage, np.uint8)]
    nat.check(nat.load().g6r_project_stage2(
        n, *[_ptr(t) for t in ins], ctypes.cast(rot9, ctypes.c_void_p), float(px), float(py),
        float(pz), float(near), float(far), float(f), float(ox), float(oy), float(lim_x),
        float(lim_y), float(width), float(height), float(low_pass), float(sh_c0), float(sh_c1),
        *[_ptr(t) for t in outs], _stream_handle()))
    for t, o in zip(outs, (means2d, conics, colors, depths, radii, stage)):
        _down(t, o)


def composite_forward(means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
                      tile_size, image, final_t, last_contrib, threads=1):
    height, width = final_t.shape
    img, ft, last = composite_arrays(means2d, conics, colors, alphas, entry_splat, tile_starts,
                                     int(tiles_x), int(tile_size), height, width, image.dtype)
    # empty tiles keep the caller's values, as in the reference kernel
    starts = np.asarray(tile_starts)
    ty_n = len(starts) - 1
    for t in range(ty_n):
        if starts[t] == starts[t + 1]:
            y0, x0 = (t // tiles_x) * tile_size, (t % tiles_x) * tile_size
            img[y0:y0 + tile_size, x0:x0 + tile_size] = image[y0:y0 + tile_size, x0:x0 + tile_size]
            ft[y0:y0 + tile_size, x0:x0 + tile_size] = final_t[y0:y0 + tile_size, x0:x0 + tile_size]
            last[y0:y0 + tile_size, x0:x0 + tile_size] = last_contrib[y0:y0 + tile_size,
                                                                      x0:x0 + tile_size]
    image[...] = img
    final_t[...] = ft
    last_contrib[...] = last


def composite_backward(means2d, conics, colors, alphas, entry_splat, tile_starts, tiles_x,
                       tile_size, final_t, last_contrib, grad_image, entry_grads, threads=1):
    height, width = final_t.shape
    tiles_y = (height + tile_size - 1) // tile_size
    m = len(np.asarray(alphas))
    ins = [_up(np.asarray(means2d).reshape(-1, 2), np.float64),
           _up(np.asarray(conics).reshape(-1, 3), np.float64),
           _up(np.asarray(colors).reshape(-1, 3), np.float64), _up(alphas, np.float64),
           _up(entry_splat, np.int32), _up(tile_starts, np.int64)]
    tail = [_up(final_t, np.float64), _up(last_contrib, np.int32), _up(grad_image, np.float64)]
    grads = _up(entry_grads, np.float64)
    nat.check(nat.load().g6r_composite_backward(
        m, *[_ptr(t) for t in ins], int(tiles_x), int(tiles_y), int(tile_size), int(width),
        int(height), *[_ptr(t) for t in tail], _ptr(grads), _stream_handle()))
    _down(grads, entry_grads)
