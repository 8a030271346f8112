"""Compositor lane-efficiency model (CPU analysis only, uses the oracle).

For one cfg3 orbit view, walks every tile's sorted run the way k_composite's
band CTAs do (16x8 bands, four 8x4 warp blocks) and counts hit-loop
iterations when each warp walks one hit list (G = 1, today), or when its lanes
are split into G groups that each walk their own list (G = 2: 4x4 quads,
4: 4x2 blocks, 8: 2x2 blocks): per 32-entry chunk a warp then iterates
max over groups of the group's hits.  Termination is ignored.

    python tools/lane_sim.py [--view 0] [--limit N]
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
from cull_stats import cull_q  # noqa: E402

GROUPS = {1: (8, 4), 2: (4, 4), 4: (4, 2), 8: (2, 2), 16: (2, 1), 32: (1, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limit", type=int, default=1_000_000)
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--size", type=int, default=512)
    args = ap.parse_args()
    scene = scenes.psi_decode_scene(limit=args.limit)
    cam = scenes.orbit_ring(scene, count=100, size=args.size)[args.view]
    prep = O.prepare(scene)
    rows = O.select_rows(scene, prep, None)[0]
    sp = O.project(scene, prep, rows, cam)
    ent = O.bin_splats(sp.means2d, sp.radii, sp.depths, args.size, args.size)
    m2 = sp.means2d.astype(np.float32).astype(np.float64)
    con = sp.conics.astype(np.float32).astype(np.float64)
    al = sp.alphas.astype(np.float32).astype(np.float64)
    qc = cull_q(al)
    a, b, c = con[:, 0], con[:, 1], con[:, 2]
    det = a * c - b * b
    with np.errstate(all="ignore"):
        ex = np.where(qc > 0, np.sqrt(np.maximum(qc, 0) * c / det) * 1.0001 + 1e-3, -1e30)
        ey = np.where(qc > 0, np.sqrt(np.maximum(qc, 0) * a / det) * 1.0001 + 1e-3, -1e30)
    es = ent.entry_splat
    starts = ent.tile_starts
    tiles_x = (args.size + 15) // 16
    tile_of = np.repeat(np.arange(len(starts) - 1), np.diff(starts))
    pos = np.arange(len(es)) - starts[tile_of]          # index inside the run
    chunk = pos // 32
    tx0 = (tile_of % tiles_x) * 16.0
    ty0 = (tile_of // tiles_x) * 16.0
    mx, my, rx, ry = m2[es, 0], m2[es, 1], ex[es], ey[es]
    print(f"view {args.view}: M={len(al)} E={len(es)} tiles={len(starts) - 1}")
    res = {}
    for G, (gw, gh) in GROUPS.items():
        iters = 0
        union = 0
        lane_slots = 0
        for wy in range(4):              # warp blocks of the 16x16 tile: 2 x 4 of 8x4
            for wx in range(2):
                hit_any = np.zeros(len(es), bool)
                per_group = []
                for gy in range(4 // gh):
                    for gx in range(8 // gw):
                        x0 = tx0 + wx * 8 + gx * gw
                        y0 = ty0 + wy * 4 + gy * gh
                        h = ((mx + rx >= x0) & (mx - rx <= x0 + gw - 1) &
                             (my + ry >= y0) & (my - ry <= y0 + gh - 1))
                        per_group.append(h)
                        hit_any |= h
                union += int(hit_any.sum())
                # per (tile, chunk): max over groups of the group's hits
                key = tile_of * 4096 + chunk
                uk, inv = np.unique(key, return_inverse=True)
                mx_g = np.zeros(len(uk), np.int64)
                for h in per_group:
                    cnt = np.bincount(inv, weights=h, minlength=len(uk)).astype(np.int64)
                    mx_g = np.maximum(mx_g, cnt)
                iters += int(mx_g.sum())
                lane_slots += sum(int(h.sum()) for h in per_group) * (32 // G)
        res[G] = iters
        print(f"G={G} ({gw}x{gh} lanes/group {32 // G}): warp iterations {iters} "
              f"(union {union}); useful group-visits x lanes / (iters x 32) = "
              f"{lane_slots / max(iters * 32, 1):.3f}; vs G=1: {iters / res[1]:.3f}")


if __name__ == "__main__":
    main()
