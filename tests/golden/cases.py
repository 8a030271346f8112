"""Fixture definitions (fine-tune loop, scene ingest) shared by make_golden.py (which runs the
reference here) and the tests (which run anywhere): inputs regenerate from
seeds, so only the reference's outputs are stored."""

import numpy as np

# (name, H, W, target channels, LossConfig kwargs); images from default_rng(700 + i)
LOSS_CASES = [
    ("single", 48, 64, 3, {}),
    ("ms5", 180, 192, 4, {}),
    ("ms3", 50, 60, 3, dict(ms_ssim_scales=3, ms_ssim_weights=(0.2, 0.5, 0.3))),
    ("l1only", 40, 44, 4, dict(lambda_ssim=0.0)),
    ("ssimonly", 176, 177, 3, dict(lambda_l1=0.0)),
]


def loss_images(seed, h, w, tc):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (h, w, 4)), rng.uniform(0.0, 1.0, (h, w, tc))


def oracle_kwargs(kw):
    """LossConfig kwargs -> oracle.loss_parts kwargs (LossConfig defaults)."""
    w = np.asarray(kw.get("ms_ssim_weights", (0.0448, 0.2856, 0.3001, 0.2363, 0.1333)), np.float64)
    return dict(lambda_l1=kw.get("lambda_l1", 0.8), lambda_ssim=kw.get("lambda_ssim", 0.2),
                scales=kw.get("ms_ssim_scales", 5), weights=tuple(w / w.sum()))


# (name, fixture scene, views [(azimuth, elevation, W, H)], iters, seed, finetune kwargs);
# view k's target is scenes.synthetic_target(W, H, seed=k)
FINETUNE_CASES = [
    ("small", "rand400", [(-0.8, 0.2, 64, 48), (0.7, -0.1, 64, 48)], 20, 3, {}),
    ("ms", "rand400", [(-0.8, 0.2, 192, 180)], 3, 4, dict(base_lr=5e-3)),
]


# Psi decode (priming.py:232-285): full-resolution dims, seed; inputs regenerate
# from default_rng(seed) via ingest_inputs
INGEST_CASES = [("identity", (22, 18, 20), 31, False), ("rotated", (17, 24, 14), 32, True)]


def ingest_inputs(dims, seed, rotated):
    """(psi (37, D/2, H/2, W/2) f64 rounded through f32, in6 channels (6, D, H, W),
    consolidated labels (D, H, W) u8 with ~30% foreground, spacing, origin, direction)."""
    rng = np.random.default_rng(seed)
    d, h, w = dims
    labels = np.where(rng.uniform(size=dims) < 0.3, rng.integers(1, 12, size=dims), 0).astype(np.uint8)
    in6 = rng.uniform(0.0, 1.0, (6,) + dims)
    in6[5] = np.clip(in6[5], 0.05, 0.95)
    psi = rng.normal(0.0, 0.3, (37, d // 2, h // 2, w // 2)).astype(np.float32).astype(np.float64)
    spacing = np.array([0.8, 1.25, 2.0])
    origin = np.array([-10.0, 3.5, 7.25])
    if rotated:
        c, s = 0.6, 0.8   # exact in binary: rotation about y with cos 0.6, sin 0.8
        direction = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
    else:
        direction = np.eye(3)
    return psi, in6, labels, spacing, origin, direction
