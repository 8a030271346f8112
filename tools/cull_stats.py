"""Compositor culling statistics on the CPU (analysis only, uses the oracle).

For one cfg3 orbit view, every (splat, warp pixel block) pair that passes the
per-warp 3-sigma box test of k_composite is classified by how many of the
block's 32 pixels actually see power in [-4.5, 0] and alpha >= 1/255, and by
whether the tighter ellipse-vs-rectangle test (min of the conic's quadratic
form over the block) would have kept it.

    python tools/cull_stats.py [--limit N] [--sample F]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_2505_17338_b200 import scenes  # noqa: E402


def cull_q(alpha):
    amax = alpha * (1 + 1e-5)
    q = 2 * np.log(np.maximum(amax * 255.0, 1e-30)) * (1 + 1e-4) + 1e-3
    return np.where(amax > 1 / 255.0, np.minimum(q, 9.0), -1.0)


def rect_min_q(a, b, c, lx, hx, ly, hy):
    """min of a x^2 + 2 b x y + c y^2 over [lx,hx] x [ly,hy] (PD form)."""
    inside = (lx <= 0) & (hx >= 0) & (ly <= 0) & (hy >= 0)
    best = np.full(a.shape, np.inf)
    for X in (lx, hx):
        y = np.clip(-b * X / c, ly, hy)
        best = np.minimum(best, a * X * X + 2 * b * X * y + c * y * y)
    for Y in (ly, hy):
        x = np.clip(-b * Y / a, lx, hx)
        best = np.minimum(best, a * x * x + 2 * b * x * Y + c * Y * Y)
    return np.where(inside, 0.0, best)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limit", type=int, default=1_000_000)
    ap.add_argument("--sample", type=float, default=0.05)
    ap.add_argument("--view", type=int, default=0)
    args = ap.parse_args()
    scene = scenes.psi_decode_scene(limit=args.limit)
    cam = scenes.orbit_ring(scene, count=100, size=512)[args.view]
    prep = O.prepare(scene)
    rows = O.select_rows(scene, prep, None)[0]
    sp = O.project(scene, prep, rows, cam)
    m2 = sp.means2d.astype(np.float32)
    con = sp.conics.astype(np.float32)
    al = sp.alphas.astype(np.float32)
    rad = sp.radii
    rng = np.random.default_rng(0)
    pick = rng.random(len(al)) < args.sample
    m2, con, al, rad = m2[pick], con[pick], al[pick], rad[pick]
    qc = cull_q(al.astype(np.float64))
    a, b, c = (con[:, k].astype(np.float64) for k in range(3))
    det = a * c - b * b
    with np.errstate(all="ignore"):
        ex = np.sqrt(np.maximum(qc, 0) * c / det) * 1.0001 + 1e-3
        ey = np.sqrt(np.maximum(qc, 0) * a / det) * 1.0001 + 1e-3
    W = H = 512
    # candidate warp blocks: 8x4 pixel blocks overlapping the splat's tile rect
    stats = {"box": 0, "ellipse": 0, "lanes_pw": 0, "lanes_alpha": 0, "zero": 0,
             "hist": np.zeros(33, np.int64)}
    pix_dx = (np.arange(32) % 8).astype(np.float32)
    pix_dy = (np.arange(32) // 8).astype(np.float32)
    for i in range(len(al)):
        if not (qc[i] > 0) or not np.isfinite(ex[i]):
            continue
        x0 = max(0, int(np.floor((m2[i, 0] - ex[i]) / 8)))
        x1 = min(W // 8 - 1, int(np.floor((m2[i, 0] + ex[i]) / 8)))
        y0 = max(0, int(np.floor((m2[i, 1] - ey[i]) / 4)))
        y1 = min(H // 4 - 1, int(np.floor((m2[i, 1] + ey[i]) / 4)))
        # restrict to the splat's binned tiles (radius rect), as the compositor does
        r = rad[i]
        tx0, tx1 = max(0, int((m2[i, 0] - r[0]) // 16)), min(31, int((m2[i, 0] + r[0]) // 16))
        ty0, ty1 = max(0, int((m2[i, 1] - r[1]) // 16)), min(31, int((m2[i, 1] + r[1]) // 16))
        x0, x1 = max(x0, tx0 * 2), min(x1, tx1 * 2 + 1)
        y0, y1 = max(y0, ty0 * 4), min(y1, ty1 * 4 + 3)
        if x0 > x1 or y0 > y1:
            continue
        bx, by = np.meshgrid(np.arange(x0, x1 + 1), np.arange(y0, y1 + 1))
        bx, by = bx.ravel(), by.ravel()
        n = bx.size
        stats["box"] += n
        lx = bx * 8 - np.float64(m2[i, 0])
        ly = by * 4 - np.float64(m2[i, 1])
        mq = rect_min_q(np.full(n, a[i]), np.full(n, b[i]), np.full(n, c[i]), lx, lx + 7, ly, ly + 3)
        keep = mq <= qc[i] * 1.0002 + 1e-6
        stats["ellipse"] += int(keep.sum())
        # octagon: the box plus the two diagonal slabs of the ellipse
        r1 = np.sqrt(qc[i] * (a[i] + c[i] - 2 * b[i]) / det[i]) * 1.0001 + 2e-3
        r2 = np.sqrt(qc[i] * (a[i] + c[i] + 2 * b[i]) / det[i]) * 1.0001 + 2e-3
        s1 = np.float64(m2[i, 0]) + np.float64(m2[i, 1])
        s2 = np.float64(m2[i, 0]) - np.float64(m2[i, 1])
        X0, Y0 = bx * 8.0, by * 4.0
        oct_keep = ((s1 + r1 >= X0 + Y0) & (s1 - r1 <= X0 + 7 + Y0 + 3) &
                    (s2 + r2 >= X0 - Y0 - 3) & (s2 - r2 <= X0 + 7 - Y0))
        stats["octagon"] = stats.get("octagon", 0) + int(oct_keep.sum())
        dx = (bx[:, None] * 8 + pix_dx[None, :]).astype(np.float32) - m2[i, 0]
        dy = (by[:, None] * 4 + pix_dy[None, :]).astype(np.float32) - m2[i, 1]
        pw = np.float32(-0.5) * (con[i, 0] * dx * dx + con[i, 2] * dy * dy) - con[i, 1] * dx * dy
        inr = (pw <= 0) & (pw >= -4.5)
        ai = al[i] * np.exp(pw)
        ok = inr & (ai >= np.float32(1 / 255))
        stats["lanes_pw"] += int(inr.sum())
        stats["lanes_alpha"] += int(ok.sum())
        cnt = ok.sum(axis=1)
        stats["zero"] += int((cnt == 0).sum())
        np.add.at(stats["hist"], cnt, 1)
        assert not (ok.any(axis=1) & ~keep).any(), "ellipse test not conservative"
        assert not (ok.any(axis=1) & ~oct_keep).any(), "octagon test not conservative"
    box = stats["box"]
    print(f"splats sampled {pick.sum()}  box pairs {box}  ellipse pairs {stats['ellipse']} "
          f"({stats['ellipse'] / box:.3f}), octagon {stats['octagon'] / box:.3f}")
    print(f"lanes with pw in range per box pair {stats['lanes_pw'] / box:.2f}, "
          f"contributing {stats['lanes_alpha'] / box:.2f}; zero-lane pairs {stats['zero'] / box:.3f}")
    print("contributing-lane histogram (fraction):",
          np.round(stats["hist"] / box, 3).tolist())


if __name__ == "__main__":
    main()
