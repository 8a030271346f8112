"""Generate the golden fixtures in tests/golden from the UNMODIFIED reference.

Run in the build container (the reference exists only there):
    python tests/golden/make_golden.py
It imports splatct from oracle/_ref (built by oracle/build_ref.sh), renders
seeded scenes with the reference's own render_with_state, and stores inputs
that are not regenerable from a seed plus every output the parity tests pin:
SplatBatch, entry_splat, tile_starts, sorted keys, image/final_t/last_contrib
(f32 and f64) and the prepared terms.  Also stores libm expf samples.
"""

import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from splatct import raster  # noqa: E402  (the reference)
from splatct.priming import Scene as RefScene  # noqa: E402

from paper_2505_17338_b200 import scenes  # noqa: E402

# (name, seed, n, camera kwargs, config kwargs, mutate)
CASES = [
    ("rand1", 0, 1, dict(azimuth=0.0, elevation=0.0, width=48, height=40), {}),
    ("rand40", 2, 40, dict(azimuth=0.6, elevation=0.3, width=48, height=40), {}),
    ("rand400", 5, 400, dict(azimuth=-0.8, elevation=0.2, width=96, height=80), {}),
    ("rand400_raw", 6, 400, dict(azimuth=1.3, elevation=-0.4, width=64, height=64),
     dict(w_mode="raw")),
    ("rand400_t8", 8, 400, dict(azimuth=2.2, elevation=0.1, width=70, height=50),
     dict(tile_size=8)),
    ("cull100", 13, 100, dict(azimuth=0.0, elevation=0.0, width=64, height=64), {}),
    ("ties50", 14, 50, dict(azimuth=2.1, elevation=0.3, width=64, height=64), {}),
    # wider sweeps (round 3): bigger scenes, steep and low poses, non-square frames
    ("rand1500_wide", 21, 1500, dict(azimuth=3.5, elevation=0.9, width=160, height=96), {}),
    ("rand2000_low", 22, 2000, dict(azimuth=-2.4, elevation=-1.0, width=112, height=128), {}),
    ("rand800_raw", 23, 800, dict(azimuth=0.3, elevation=0.5, width=100, height=140),
     dict(w_mode="raw")),
]


def to_ref(s):
    return RefScene(mu_p=s.mu_p, mu_d=s.mu_d, cov_raw=s.cov_raw, sh=s.sh,
                    opacity_raw=s.opacity_raw, labels=s.labels, spacing=s.spacing,
                    origin=s.origin, direction=s.direction, spatial_scale=s.spatial_scale,
                    directional_scale=s.directional_scale)


def make_case(name, seed, n, cam_kw, cfg_kw):
    rng = np.random.default_rng(seed)
    box = 8.0 if name.startswith("ties") else 22.0
    s = scenes.random_scene(rng, n, box=box, iso=name.startswith("ties"))
    cam = scenes.orbit_camera(**cam_kw)
    if name.startswith("cull"):
        mu = s.mu_p.copy()
        mu[5] = (0.0, 0.0, 200.0)
        mu[6] = (900.0, 0.0, 0.0)
        mu[8] = cam.position
        op = s.opacity_raw.copy()
        op[12] = -9.0
        s = s.with_params(mu_p=mu, opacity_raw=op)
    if name.startswith("ties"):
        mu = s.mu_p.copy()
        mu[1] = mu[0]
        mu[3] = mu[2] * (1.0 + 1e-12)
        mu[10:15] = mu[10]
        s = s.with_params(mu_p=mu)
    out = dict(mu_p=s.mu_p, mu_d=s.mu_d, cov_raw=s.cov_raw, sh=s.sh, opacity_raw=s.opacity_raw,
               labels=s.labels, spatial_scale=s.spatial_scale,
               directional_scale=np.float64(s.directional_scale),
               cam_position=cam.position, cam_rotation=cam.rotation,
               cam_fov=np.float64(cam.fov_y), cam_wh=np.array([cam.width, cam.height]))
    rs = to_ref(s)
    for prec in ("f32", "f64"):
        cfg = raster.RenderConfig(precision=prec, threads=1, **cfg_kw)
        st = raster.render_with_state(rs, cam, None, cfg)
        out[f"{prec}_image"] = st.image
        out[f"{prec}_final_t"] = st.final_t
        out[f"{prec}_last_contrib"] = st.last_contrib
    sp = st.splats
    for f in ("gids", "means2d", "conics", "colors", "alphas", "depths", "radii"):
        out[f"splat_{f}"] = getattr(sp, f)
    out["entry_splat"] = st.entries.entry_splat
    out["tile_starts"] = st.entries.tile_starts
    out["stats"] = np.array([st.stats.n_drawn, st.stats.n_entries, st.stats.n_view_degenerate,
                             st.stats.n_alpha_culled, st.stats.n_depth_culled,
                             st.stats.n_projection_culled, st.stats.n_viewport_culled])
    prep = raster.prepare_scene(rs, cfg_kw.get("w_mode", "peak"))
    for f in ("adjust", "precision_dd", "sigma_prime", "w_norm", "degenerate"):
        out[f"prep_{f}"] = getattr(prep.terms, f)
    out["prep_opacity"] = prep.opacity
    out["config"] = np.array([cfg_kw.get("tile_size", 16), 1 if cfg_kw.get("w_mode") == "raw" else 0])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "M", st.stats.n_drawn, "E", st.stats.n_entries)


BACKWARD_CASES = ("rand40", "rand400", "rand400_raw", "cull100", "rand1500_wide", "rand2000_low",
                  "rand800_raw")


def make_backward(name):
    """Reference render_backward (diffrender.py:401-439) for a fixture scene and
    a seeded d loss / d image."""
    from splatct.diffrender import render_backward
    z = np.load(os.path.join(HERE, f"{name}.npz"))
    s = RefScene(mu_p=z["mu_p"], mu_d=z["mu_d"], cov_raw=z["cov_raw"], sh=z["sh"],
                 opacity_raw=z["opacity_raw"], labels=z["labels"], spacing=np.ones(3),
                 origin=np.zeros(3), direction=np.eye(3), spatial_scale=z["spatial_scale"],
                 directional_scale=float(z["directional_scale"]))
    from splatct.camera import Camera
    w, h = (int(v) for v in z["cam_wh"])
    cam = Camera(position=z["cam_position"], rotation=z["cam_rotation"], fov_y=float(z["cam_fov"]),
                 width=w, height=h)
    w_mode = "raw" if int(z["config"][1]) else "peak"
    g = np.random.default_rng(1000 + len(name)).normal(size=(h, w, 4))
    buf = render_backward(s, cam, g, None, raster.RenderConfig(precision="f64", w_mode=w_mode,
                                                               threads=1))
    np.savez_compressed(os.path.join(HERE, f"bwd_{name}.npz"), grad_image=g,
                        **{f"g_{k}": getattr(buf, k) for k in
                           ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw")})
    print("bwd", name, float(np.abs(buf.cov_raw).max()))


def make_expf():
    libm = ctypes.CDLL("libm.so.6")
    libm.expf.restype = ctypes.c_float
    libm.expf.argtypes = [ctypes.c_float]
    rng = np.random.default_rng(123)
    x = np.concatenate([rng.uniform(-4.5, 0.0, 20000), -np.logspace(-8, np.log10(4.5), 2000),
                        np.array([0.0, -4.5, -1e-30, -0.5, -1.0])]).astype(np.float32)
    y = np.array([libm.expf(float(v)) for v in x], dtype=np.float32)
    np.savez_compressed(os.path.join(HERE, "expf_glibc.npz"), x=x, y=y)


from cases import FINETUNE_CASES, INGEST_CASES, LOSS_CASES, ingest_inputs, loss_images  # noqa: E402


def make_loss():
    """Reference _loss_parts (diffrender.py:117-138) on seeded images; stores
    the scalars, the full gradient for small cases and a seeded sample of
    gradient entries plus per-channel sums for the large ones."""
    from splatct.diffrender import LossConfig, _loss_parts
    out = {}
    for i, (name, h, w, tc, kw) in enumerate(LOSS_CASES):
        p, g = loss_images(700 + i, h, w, tc)
        total, l1, ssim_loss, grad = _loss_parts(p, g, LossConfig(**kw))
        idx = np.random.default_rng(900 + i).choice(grad.size, min(grad.size, 4096), replace=False)
        out[f"{name}_parts"] = np.array([total, l1, ssim_loss])
        out[f"{name}_idx"] = idx
        out[f"{name}_grad_sample"] = grad.reshape(-1)[idx]
        out[f"{name}_grad_sums"] = grad.sum(axis=(0, 1))
        out[f"{name}_grad_abs"] = np.abs(grad).sum(axis=(0, 1))
        print("loss", name, total, l1, ssim_loss)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **out)


def make_finetune():
    """Reference finetune (diffrender.py:548-585) on a fixture scene against
    synthetic_target views: history rows and the final parameters."""
    from splatct.diffrender import finetune
    for name, fixture, views, iters, seed, kw in FINETUNE_CASES:
        z = np.load(os.path.join(HERE, f"{fixture}.npz"))
        s = RefScene(mu_p=z["mu_p"], mu_d=z["mu_d"], cov_raw=z["cov_raw"], sh=z["sh"],
                     opacity_raw=z["opacity_raw"], labels=z["labels"], spacing=np.ones(3),
                     origin=np.zeros(3), direction=np.eye(3), spatial_scale=z["spatial_scale"],
                     directional_scale=float(z["directional_scale"]))
        pairs = []
        for k, (az, el, w, h) in enumerate(views):
            cam = scenes.orbit_camera(azimuth=az, elevation=el, width=w, height=h)
            pairs.append((cam, scenes.synthetic_target(w, h, seed=k)))
        out, hist = finetune(s, pairs, iters=iters, seed=seed, **kw)
        np.savez_compressed(
            os.path.join(HERE, f"ft_{name}.npz"),
            history=np.array([[r["iteration"], r["lr"], r["l1"], r["ssim_loss"], r["total"]]
                              for r in hist]),
            **{k: getattr(out, k) for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw")})
        print("finetune", name, hist[-1])


def make_ingest():
    """Reference decode_param_volume (priming.py:232-285) on seeded volumes."""
    from splatct.priming import ParamVolume, decode_param_volume
    from splatct.volume import InputVolume6, LabelVolume
    for name, dims, seed, rotated in INGEST_CASES:
        psi, in6, labels, spacing, origin, direction = ingest_inputs(dims, seed, rotated)
        s = decode_param_volume(ParamVolume(psi), InputVolume6(in6, spacing, origin, direction),
                                LabelVolume(labels, consolidated=True))
        np.savez_compressed(os.path.join(HERE, f"ingest_{name}.npz"),
                            **{k: getattr(s, k) for k in ("mu_p", "mu_d", "cov_raw", "sh",
                                                          "opacity_raw", "labels",
                                                          "spatial_scale")})
        print("ingest", name, len(s))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ingest":
        make_ingest()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "train":
        make_loss()
        make_finetune()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "cases":   # only the named cases (+ their backward)
        for case in CASES:
            if case[0] in sys.argv[2:]:
                make_case(*case)
                if case[0] in BACKWARD_CASES:
                    make_backward(case[0])
        sys.exit(0)
    only_bwd = len(sys.argv) > 1 and sys.argv[1] == "backward"
    if not only_bwd:
        for case in CASES:
            make_case(*case)
        make_expf()
    for name in BACKWARD_CASES:
        make_backward(name)
