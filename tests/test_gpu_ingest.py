"""Scene ingest on the device against the reference:
Psi decode (priming.py:232-285) vs golden vectors from the unmodified
reference (tests/golden/make_golden.py ingest), the .meta/.raw file path, and
the group filter (priming.py:362-374) vs the host filter.  Integer/byte work
and IEEE basic ops: bit-exact."""

import os

import numpy as np
import pytest

from paper_2505_17338_b200 import ingest, scenes
from paper_2505_17338_b200.errors import EmptySceneError, VolumeFormatError
from paper_2505_17338_b200.multigpu import DeviceScene
from paper_2505_17338_b200.scene import filter_scene

from cases import INGEST_CASES, ingest_inputs
from test_oracle import GOLDEN

pytestmark = pytest.mark.gpu


class _Vol:   # duck-typed InputVolume6 / LabelVolume
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _inputs(dims, seed, rotated):
    psi, in6, labels, spacing, origin, direction = ingest_inputs(dims, seed, rotated)
    return (ingest.ParamVolume(psi),
            _Vol(channels=in6, spacing=spacing, origin=origin, direction=direction),
            _Vol(labels=labels, consolidated=True))


@pytest.mark.parametrize("case", INGEST_CASES, ids=[c[0] for c in INGEST_CASES])
def test_psi_decode_matches_reference_golden(case):
    name, dims, seed, rotated = case
    z = np.load(os.path.join(GOLDEN, f"ingest_{name}.npz"))
    s = ingest.decode_param_volume(*_inputs(dims, seed, rotated))
    for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels", "spatial_scale"):
        np.testing.assert_array_equal(getattr(s, k), z[k], err_msg=k)


def test_psi_decode_from_f32_files_matches_f64_path(tmp_path):
    name, dims, seed, rotated = INGEST_CASES[0]
    psi, in6, labels = _inputs(dims, seed, rotated)
    ingest.save_param_volume(psi, tmp_path / "psi")
    loaded = ingest.load_param_volume(tmp_path / "psi")
    assert loaded.channels.dtype == np.float32
    a = ingest.decode_param_volume_device(loaded, in6, labels)
    b = ingest.decode_param_volume_device(psi, in6, labels)
    for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
        assert bool((getattr(a, k) == getattr(b, k)).all()), k


def test_psi_decode_validation():
    name, dims, seed, rotated = INGEST_CASES[0]
    psi, in6, labels = _inputs(dims, seed, rotated)
    with pytest.raises(VolumeFormatError):
        ingest.decode_param_volume(ingest.ParamVolume(psi.channels[:, :-1]), in6, labels)
    empty = _Vol(labels=np.zeros_like(labels.labels), consolidated=True)
    with pytest.raises(EmptySceneError):
        ingest.decode_param_volume(psi, in6, empty)


def test_psi_decode_large_grid_matches_oracle(oracle):
    """A 160x150x140 volume (420k half-grid voxels in 103 chunks, ~126k rows)
    against the oracle's numpy restatement: bit-exact."""
    psi, in6, labels = _inputs((160, 150, 140), 77, True)
    got = ingest.decode_param_volume(psi, in6, labels)
    want = oracle.decode_param_volume(psi.channels, in6.channels, labels.labels, in6.spacing,
                                      in6.origin, in6.direction)
    for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
        np.testing.assert_array_equal(getattr(got, k), want[k], err_msg=k)


def test_group_filter_on_device_matches_host_filter():
    s = scenes.random_scene(np.random.default_rng(21), 30000)
    dev = DeviceScene(*[__import__("torch").from_numpy(np.ascontiguousarray(getattr(s, k))).cuda()
                        for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels")],
                      spatial_scale=s.spatial_scale, directional_scale=s.directional_scale)
    for mask in ([2, 5, 7], [], list(range(12)), [11]):
        want = filter_scene(s, mask)
        got = ingest.filter_scene_device(dev, mask)
        assert len(got) == len(want)
        for k in ("mu_p", "mu_d", "cov_raw", "sh", "opacity_raw", "labels"):
            np.testing.assert_array_equal(getattr(got, k).cpu().numpy(), getattr(want, k))
