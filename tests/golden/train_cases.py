"""Fine-tune loop fixture definitions shared by make_golden.py (which runs the
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
