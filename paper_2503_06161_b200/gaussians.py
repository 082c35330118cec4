"""Host-side types of the render path: GaussianCloud, CameraFrame, activations.

API mirror of featsplat.gaussians (gaussians.py:25-133, 298-302).  These are
plain containers of float64 NumPy arrays exactly like the reference, so user
code constructing clouds and frames does not change; the math that consumes
them runs in libfs4d (sm_100a).

Extension: ``GaussianCloud.sh_rest`` ([K, (L+1)^2-1, 3], default None) holds
spherical-harmonic bands above degree 0; degree 0 is ``colors_raw`` as in the
reference (see csrc/sh.cuh).
"""

from dataclasses import dataclass

import numpy as np

from .errors import DataError, DegenerateRotationError, NumericalError

_PARAM_FIELDS = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw",
                 "features")


def sigmoid(x):
    """Numerically stable logistic (gaussians.py:25-31 semantics)."""
    x = np.asarray(x, dtype=np.float64)
    z = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + z), z / (1.0 + z))


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass
class GaussianCloud:
    """Struct-of-arrays cloud of K Gaussians with N semantic channels."""

    positions: np.ndarray       # [K, 3]
    rotations: np.ndarray       # [K, 4] raw (w, x, y, z)
    log_scales: np.ndarray      # [K, 3]
    opacity_logits: np.ndarray  # [K]
    colors_raw: np.ndarray      # [K, 3] (SH degree-0 term)
    features: np.ndarray        # [K, N]
    sh_rest: np.ndarray = None  # [K, (L+1)^2-1, 3] or None (build extension)

    def __len__(self):
        return int(np.shape(self.positions)[0])

    @property
    def feature_dim(self):
        return int(np.shape(self.features)[1])

    @property
    def sh_degree(self):
        if self.sh_rest is None or np.shape(self.sh_rest)[1] == 0:
            return 0
        return int(round(np.sqrt(np.shape(self.sh_rest)[1] + 1))) - 1

    def scales(self):
        return np.exp(self.log_scales)

    def opacities(self):
        return sigmoid(self.opacity_logits)

    def colors(self):
        return np.clip(self.colors_raw, 0.0, 1.0)

    def unit_rotations(self):
        n = np.sqrt(np.sum(np.square(self.rotations), axis=1, keepdims=True))
        if np.any(n < 1e-12):
            raise DegenerateRotationError("quaternion norm below 1e-12")
        return self.rotations / n

    def validate(self):
        for name in _PARAM_FIELDS:
            if not np.isfinite(getattr(self, name)).all():
                raise NumericalError(f"non-finite entries in cloud.{name}")
        self.unit_rotations()

    def copy(self):
        return GaussianCloud(*(np.array(getattr(self, f), copy=True) for f in _PARAM_FIELDS),
                             sh_rest=None if self.sh_rest is None else np.array(self.sh_rest))

    def param_arrays(self):
        out = {name: getattr(self, name) for name in _PARAM_FIELDS}
        if self.sh_rest is not None:
            out["sh_rest"] = self.sh_rest
        return out


@dataclass
class CameraFrame:
    """One posed frame; only K, T, time and the image size feed the render path."""

    K: np.ndarray
    T: np.ndarray
    time: float
    image: np.ndarray
    depth: np.ndarray
    mask: np.ndarray
    features: object = None
    labels: np.ndarray = None

    def __post_init__(self):
        # validation rules of gaussians.py:110-125
        K = np.array(self.K, dtype=np.float64)
        if K.shape != (3, 3) or not (K[0, 0] > 0 and K[1, 1] > 0):
            raise DataError("intrinsics must be 3x3 with positive focal lengths")
        if abs(np.linalg.det(K)) < 1e-12:
            raise DataError("intrinsics matrix is singular")
        T = np.array(self.T, dtype=np.float64)
        rot = T[:3, :3]
        if np.abs(rot.T @ rot - np.eye(3)).max() > 1e-6:
            raise DataError("extrinsics rotation block is not orthonormal")
        if np.shape(self.depth) != np.shape(self.mask):
            raise DataError("depth and mask shapes differ")
        if np.any(np.asarray(self.depth)[np.asarray(self.mask, dtype=bool)] < 0):
            raise DataError("negative depth inside mask")
        self.K, self.T = K, T

    @property
    def height(self):
        return int(np.shape(self.image)[0])

    @property
    def width(self):
        return int(np.shape(self.image)[1])


def scene_aabb(cloud, pad=0.05):
    """Padded bounding box of the positions (gaussians.py:298-302)."""
    p = np.asarray(cloud.positions, dtype=np.float64)
    lo, hi = p.min(axis=0), p.max(axis=0)
    span = np.maximum(hi - lo, 1e-6)
    return np.stack([lo - pad * span, hi + pad * span])
