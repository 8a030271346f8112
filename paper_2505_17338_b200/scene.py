"""Scene container: the render path's Gaussian input contract.

Same structure-of-arrays as the reference ``Scene`` (priming.py:50-122):
float64 ``mu_p (N,3)``, ``mu_d (N,3)``, ``cov_raw (N,21)``, ``sh (N,12)``,
``opacity_raw (N)``, ``labels (N) uint8`` in [1, 11], plus ``spatial_scale
(3)`` and ``directional_scale``.  Identity-keyed (``eq=False``) so the device
copy and prepared terms can be cached per instance.  The renderer accepts any
object with these attributes, including the reference's own ``Scene``.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .errors import InvalidParameterError

N_GROUPS = 12
N_COV_RAW = 21
N_SH = 12


@dataclass(frozen=True, eq=False)
class Scene:
    mu_p: np.ndarray
    mu_d: np.ndarray
    cov_raw: np.ndarray
    sh: np.ndarray
    opacity_raw: np.ndarray
    labels: np.ndarray
    spacing: np.ndarray = None
    origin: np.ndarray = None
    direction: np.ndarray = None
    spatial_scale: np.ndarray = None
    directional_scale: float = 1.0

    def __post_init__(self):
        n = len(self.mu_p)
        for name, shape in (("mu_p", (n, 3)), ("mu_d", (n, 3)), ("cov_raw", (n, N_COV_RAW)),
                            ("sh", (n, N_SH)), ("opacity_raw", (n,))):
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
            if arr.shape != shape:
                raise InvalidParameterError(f"{name} must have shape {shape}, got {arr.shape}")
            if not np.all(np.isfinite(arr)):
                raise InvalidParameterError(f"{name} contains non-finite values")
            object.__setattr__(self, name, arr)
        labels = np.ascontiguousarray(self.labels)
        if labels.shape != (n,):
            raise InvalidParameterError(f"labels must have shape ({n},)")
        if n and (labels.min() < 1 or labels.max() >= N_GROUPS):
            raise InvalidParameterError(f"scene labels must lie in [1, {N_GROUPS - 1}]")
        object.__setattr__(self, "labels", labels.astype(np.uint8))
        for name, shape, default in (("spacing", (3,), np.ones(3)), ("origin", (3,), np.zeros(3)),
                                     ("direction", (3, 3), np.eye(3)),
                                     ("spatial_scale", (3,), np.ones(3))):
            val = getattr(self, name)
            arr = np.asarray(default if val is None else val, dtype=np.float64)
            if name == "spatial_scale" and arr.shape == ():
                arr = np.full(3, float(arr))
            if arr.shape != shape or not np.all(np.isfinite(arr)):
                raise InvalidParameterError(f"{name} must be a finite array of shape {shape}")
            object.__setattr__(self, name, arr)
        object.__setattr__(self, "directional_scale", float(self.directional_scale))

    def __len__(self) -> int:
        return self.mu_p.shape[0]

    @property
    def group_counts(self) -> np.ndarray:
        return np.bincount(self.labels, minlength=N_GROUPS)

    def take(self, indices) -> "Scene":
        return replace(self, mu_p=self.mu_p[indices], mu_d=self.mu_d[indices],
                       cov_raw=self.cov_raw[indices], sh=self.sh[indices],
                       opacity_raw=self.opacity_raw[indices], labels=self.labels[indices])

    def with_params(self, **arrays) -> "Scene":
        return replace(self, **arrays)


def filter_scene(scene, group_mask) -> "Scene":
    """Rows whose label is in ``group_mask`` (priming.py:362-374)."""
    groups = np.zeros(N_GROUPS, dtype=bool)
    for g in group_mask:
        if not 0 <= int(g) < N_GROUPS:
            raise InvalidParameterError(f"group index {g} outside [0, 11]")
        groups[int(g)] = True
    return scene.take(np.nonzero(groups[scene.labels])[0])
