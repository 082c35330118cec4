"""HexPlane field (hexplane.py:16-222 API).

Planes are stored channel-last [Ra, Rb, C] float64 on the host like the
reference.  The query (bilinear gather + six-plane product) and its backward
run in libfs4d: fused into the deformation kernels on the frame path, and on
their own behind ``query`` / ``query_with_cache`` / ``query_backward``
(fs4d_hexplane_query / fs4d_hexplane_query_backward), which keep the
reference's signatures, NumPy in / out, and also accept fp32 CUDA tensors.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, ContractViolation

PLANE_AXES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
TIME_AXIS = 3


@dataclass
class HexPlaneConfig:
    levels: tuple = (1, 2, 4, 8)
    base_resolution: tuple = (64, 64, 64, 100)
    out_dim: int = 64
    feat_dim: int = 0
    init_scale: float = 0.1

    def channels_per_level(self):
        if self.feat_dim > 0:
            return self.feat_dim
        n = len(self.levels)
        if self.out_dim % n:
            raise ConfigurationError(
                f"out_dim {self.out_dim} not divisible by {n} levels; set feat_dim explicitly")
        return self.out_dim // n


def plane_shape(cfg, mult, axes):
    """Spatial axes scale with the level multiplier, time does not (hexplane.py:41-46)."""
    return tuple(cfg.base_resolution[a] * (1 if a == TIME_AXIS else mult) for a in axes)


class HexPlaneField:
    """Grids of every level plus the aabb normalising query positions."""

    def __init__(self, cfg, aabb, rng, init="reference"):
        self.cfg = cfg
        self.aabb = np.asarray(aabb, dtype=np.float64)
        if self.aabb.shape != (2, 3) or not np.all(self.aabb[1] > self.aabb[0]):
            raise ConfigurationError("aabb must be [2, 3] with hi > lo")
        self.channels = cfg.channels_per_level()
        self.planes = []
        for mult in cfg.levels:
            level = []
            for axes in PLANE_AXES:
                ra, rb = plane_shape(cfg, mult, axes)
                if min(ra, rb) < 2:
                    raise ConfigurationError("plane resolutions must be >= 2")
                shape = (ra, rb, self.channels)
                if init == "reference":   # 1 +- init_scale (hexplane.py:65-66)
                    level.append(1.0 + rng.uniform(-cfg.init_scale, cfg.init_scale, size=shape))
                elif init == "uniform":   # BASELINE configs: U[0.1, 0.5]
                    level.append(rng.uniform(0.1, 0.5, size=shape))
                elif init == "zeros":
                    level.append(np.zeros(shape))
                else:
                    raise ConfigurationError(f"unknown plane init {init!r}")
            self.planes.append(level)

    @property
    def latent_dim(self):
        return self.channels * len(self.cfg.levels)

    def normalized_coords(self, positions, t):
        """(coords [K, 4], inside [K, 3]) of hexplane.py:84-92: spatial
        coordinates (p - lo) / (hi - lo) clipped to [0, 1], inside = strictly
        within (0, 1) per axis, t clipped to [0, 1].  A host helper of the
        container (like scene_aabb); the kernels compute the same values in
        fp64 per Gaussian."""
        p = np.asarray(positions, dtype=np.float64)
        lo, hi = self.aabb[0], self.aabb[1]
        raw = (p - lo) / (hi - lo)
        coords = np.empty((p.shape[0], 4))
        coords[:, :3] = np.clip(raw, 0.0, 1.0)
        coords[:, 3] = min(max(float(t), 0.0), 1.0)
        return coords, (raw > 0.0) & (raw < 1.0)

    def param_arrays(self):
        return {f"grid.l{li}.p{pi}": plane
                for li, level in enumerate(self.planes) for pi, plane in enumerate(level)}

    def set_param(self, name, arr):
        _, l, p = name.split(".")
        self.planes[int(l[1:])][int(p[1:])] = arr


# ---------------------------------------------------------------------------
# query / query_with_cache / query_backward (hexplane.py:113-187), on device
# ---------------------------------------------------------------------------
def query(field, positions, t):
    """Latent [K, channels * levels] of `positions` at time t."""
    f, _ = query_with_cache(field, positions, t)
    return f


def query_with_cache(field, positions, t):
    """Latent plus the record query_backward needs (the device positions and
    t: the backward re-selects every bilinear cell in fp64 instead of storing
    them)."""
    import torch

    from . import _native as N
    from .device import _p, _stream, as_device, to_host
    dev, _ = _device_field(field)
    pos, host = as_device(positions)
    pos = pos.reshape(-1, 3)
    k = int(pos.shape[0])
    lat = torch.empty(k, dev.latent_dim, dtype=torch.float32, device=pos.device)
    import ctypes
    fs = dev.struct()
    N.check(N.load().fs4d_hexplane_query(ctypes.byref(fs), _p(pos), k, float(t), _p(lat), _stream()))
    cache = {"k": k, "t": float(t), "positions": pos, "field": dev, "host": host}
    return to_host(lat, host), cache


def query_backward(field, cache, dL_df):
    """(plane_grads mirroring field.planes, dL/dpositions [K, 3]); position
    gradients are zero on every clamped axis (hexplane.py:186)."""
    import torch

    from . import _native as N
    from .device import _p, _stream, as_device, to_host
    k = cache["k"]
    dev = cache.get("field") or _device_field(field)[0]
    up, _ = as_device(dL_df)
    if tuple(up.shape) != (k, dev.latent_dim):
        raise ContractViolation(f"dL_df shape {tuple(up.shape)} does not match ({k}, {dev.latent_dim})")
    grads = dev.zeros_like()
    dpos = torch.empty(k, 3, dtype=torch.float32, device=up.device)
    import ctypes
    gs, fs = grads.struct(), dev.struct()
    N.check(N.load().fs4d_hexplane_query_backward(ctypes.byref(fs), _p(cache["positions"]), k, cache["t"], _p(up),
                                                  ctypes.byref(gs), _p(dpos), 0, _stream()))
    host = cache.get("host", True)
    planes = grads.planes if not host else [[p.cpu().numpy().astype(np.float64) for p in lv] for lv in grads.planes]
    return planes, to_host(dpos, host)


# ---------------------------------------------------------------------------
# total-variation regulariser (hexplane.py:190-222), on device
# ---------------------------------------------------------------------------
def tv_loss_grad_device(field, grads=None, scale=1.0, accumulate=False, loss=None):
    """fs4d_tv_loss_grad on a DeviceField: adds scale * tv to `loss` (device
    float64 [1], optional) and writes / accumulates d(scale*tv)/d(plane) into
    `grads` (DeviceField, optional), in one pass."""
    import ctypes

    from . import _native as N
    from .device import _p, _stream

    fs = field.struct()
    gs = grads.struct() if grads is not None else None
    N.check(N.load().fs4d_tv_loss_grad(ctypes.byref(fs), ctypes.byref(gs) if gs is not None else None,
                                       float(scale), int(bool(accumulate)), _p(loss), _stream()))


def _device_field(field):
    from .device import DeviceField
    if isinstance(field, DeviceField):
        return field, False
    return DeviceField.from_field(field), True


def tv_loss(field):
    """Mean squared difference of axis-adjacent cells, summed over planes
    (hexplane.py:190-196)."""
    import torch

    dev, _ = _device_field(field)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    tv_loss_grad_device(dev, None, 1.0, False, loss)
    return float(loss.item())


def tv_backward(field, scale=1.0):
    """d(scale * tv_loss)/d(plane) for every plane (hexplane.py:207-222)."""
    dev, host = _device_field(field)
    grads = dev.zeros_like()
    tv_loss_grad_device(dev, grads, scale, False, None)
    if not host:
        return grads.planes
    return [[p.cpu().numpy().astype(np.float64) for p in level] for level in grads.planes]
