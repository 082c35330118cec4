"""Adaptive density control on device (gaussians.py:309-425) -- SURVEY §8(f)
row 4.  API mirror of the reference's ViewspaceGradStats,
DensityControlConfig, densify_and_prune, prune_only and reset_opacity.

The classification (fp64, the reference's thresholds) and the stream
compaction into the reference's row order run in libfs4d
(csrc/density.cu).  The only host work is drawing the split samples with the
caller's own ``numpy.random.Generator`` -- ``rng.standard_normal((n_split,
3))`` twice, exactly the reference's calls -- so the random stream, and with
it the split children, match the reference's.

Functions take the reference's NumPy cloud (and return / mutate NumPy like
the reference) or a DeviceCloud (device tensors, ``DeviceDensity``).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import DeviceCloud, StatusBlock, _p, _stream
from .errors import ConfigurationError


@dataclass
class DensityControlConfig:
    """gaussians.py:330-334."""

    grad_threshold: float = 2e-4
    percent_dense: float = 0.01
    prune_opacity: float = 0.005
    split_factor: float = 1.6


class ViewspaceGradStats:
    """Accumulated screen-space positional gradient norms per Gaussian
    (gaussians.py:309-327).  accum / count are float64 NumPy arrays or CUDA
    tensors; add() accumulates render_backward's viewspace_index /
    viewspace_norm (device arrays: fs4d_grad_stats_add, no host round trip)."""

    def __init__(self, accum, count):
        self.accum, self.count = accum, count

    @classmethod
    def zeros(cls, k, device=None):
        if device is None:
            return cls(accum=np.zeros(k), count=np.zeros(k))
        f = dict(dtype=torch.float64, device=device)
        return cls(accum=torch.zeros(k, **f), count=torch.zeros(k, **f))

    def add(self, indices, norms, n_dev=None):
        """accum[indices] += norms, count[indices] += 1 on the device
        (fs4d_grad_stats_add); host (NumPy) statistics are staged through the
        device and written back, so both forms run the same kernel."""
        host = not isinstance(self.accum, torch.Tensor)
        accum = torch.as_tensor(np.asarray(self.accum, np.float64), device="cuda") if host else self.accum
        count = torch.as_tensor(np.asarray(self.count, np.float64), device="cuda") if host else self.count
        idx = torch.as_tensor(np.asarray(indices) if host else indices, device=accum.device).to(torch.int32).contiguous()
        nrm = torch.as_tensor(np.asarray(norms) if host else norms, device=accum.device).to(torch.float32).contiguous()
        N.check(N.load().fs4d_grad_stats_add(_p(accum), _p(count), _p(idx), _p(nrm), idx.numel(), _p(n_dev),
                                             _stream()))
        if host:
            self.accum = accum.cpu().numpy()
            self.count = count.cpu().numpy()

    def add_dense(self, norms):
        """Accumulate render_backward's dense per-Gaussian norms (negative =
        culled) -- the source-order form the training step produces."""
        nrm = norms.to(torch.float32).contiguous()
        N.check(N.load().fs4d_grad_stats_add(_p(self.accum), _p(self.count), None, _p(nrm), nrm.numel(), None,
                                             _stream()))

    def averages(self):
        if isinstance(self.accum, torch.Tensor):
            return self.accum / torch.clamp(self.count, min=1.0)
        return self.accum / np.maximum(self.count, 1.0)


def _cfg_struct(cfg, extent):
    c = N.DensityConfig()
    c.grad_threshold, c.percent_dense = float(cfg.grad_threshold), float(cfg.percent_dense)
    c.prune_opacity, c.split_factor, c.extent = float(cfg.prune_opacity), float(cfg.split_factor), float(extent)
    return c


class DeviceDensity:
    """Two-step device density control over a DeviceCloud.

    run() classifies, reads back the four counts (the one host sync: the new
    size must be known to allocate), draws the split samples from `rng`, and
    compacts the cloud, the grad stats and any per-row extra arrays (Adam
    moments) into freshly allocated tensors."""

    def __init__(self, device="cuda"):
        self.device = device
        self.ws = None
        self.counts = torch.zeros(4, dtype=torch.int32, device=device)
        self.status = StatusBlock(device)

    def run(self, cloud, stats, cfg, extent, rng=None, prune_only=False, extras=()):
        lib = N.load()
        k = len(cloud)
        cap = 2 * k + 1
        need = int(lib.fs4d_density_workspace_bytes(k, cap))
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(max(need, 1), dtype=torch.uint8, device=self.device)
        c = _cfg_struct(cfg, extent)
        self.status.reset()
        cs = cloud.struct()
        acc = stats.accum if stats is not None else None
        cnt = stats.count if stats is not None else None
        N.check(lib.fs4d_density_classify(ctypes.byref(cs), _p(acc), _p(cnt), ctypes.byref(c), int(prune_only), cap,
                                          _p(self.counts), _p(self.ws), self.ws.numel(), _p(self.status.t),
                                          _stream()))
        n_keep, n_clone, n_split, n_out = (int(v) for v in self.counts.cpu().tolist())
        self.status.raise_if_error()
        normals = None
        if n_split:
            if rng is None:
                raise ConfigurationError("densify_and_prune needs the rng for split samples")
            z = np.stack([rng.standard_normal((n_split, 3)) for _ in range(2)])  # gaussians.py:383-384
            normals = torch.as_tensor(z, dtype=torch.float64, device=self.device).contiguous()
        out = DeviceCloud.empty(n_out, cloud.feature_dim, cloud.sh_degree, self.device)
        os_ = out.struct()
        new_stats = None
        if stats is not None:
            new_stats = ViewspaceGradStats.zeros(n_out, self.device)
        extras = list(extras)
        outs = [torch.empty((n_out,) + tuple(e.shape[1:]), dtype=torch.float32, device=self.device) for e in extras]
        n_ex = len(extras)
        ein = (ctypes.c_void_p * max(n_ex, 1))(*[e.data_ptr() for e in extras])
        eout = (ctypes.c_void_p * max(n_ex, 1))(*[o.data_ptr() for o in outs])
        ew = (ctypes.c_int32 * max(n_ex, 1))(*[int(np.prod(e.shape[1:])) if e.dim() > 1 else 1 for e in extras])
        N.check(lib.fs4d_density_apply(ctypes.byref(cs), _p(normals), ctypes.byref(c), cap, n_keep, n_clone, n_split,
                                       ctypes.byref(os_), _p(acc), _p(cnt),
                                       _p(new_stats.accum) if new_stats else None,
                                       _p(new_stats.count) if new_stats else None, int(not prune_only), n_ex, ein, eout,
                                       ew, _p(self.ws), self.ws.numel(), _p(self.status.t), _stream()))
        self.status.raise_if_error()
        report = {"cloned": n_clone, "split": n_split, "pruned": k - n_keep - n_split if not prune_only else k - n_keep,
                  "count": n_out}
        return out, new_stats, outs, report


def _host_cloud_to_device(cloud):
    return DeviceCloud.from_cloud(cloud)


def _device_to_host_cloud(dev, like):
    for name in DeviceCloud.FIELDS:
        setattr(like, name, getattr(dev, name).cpu().numpy().astype(np.float64))
    if getattr(like, "sh_rest", None) is not None and dev.sh_rest is not None:
        like.sh_rest = dev.sh_rest.cpu().numpy().astype(np.float64)


def _n_pruned(cloud, cfg):
    from .gaussians import sigmoid
    return int(np.count_nonzero(sigmoid(np.asarray(cloud.opacity_logits, dtype=np.float64)) < cfg.prune_opacity))


def densify_and_prune(cloud, grad_stats, iteration, cfg, extent, rng, adam_states=None):
    """Clone small / split large high-gradient Gaussians, prune transparent
    ones (gaussians.py:349-405).  Mutates the cloud, the gradient stats (reset
    to the new size) and the per-row Adam moment buffers if given; returns
    the reference's report dict."""
    n_pruned = _n_pruned(cloud, cfg)
    dev = _host_cloud_to_device(cloud)
    stats = ViewspaceGradStats(torch.as_tensor(np.asarray(grad_stats.accum, np.float64), device="cuda"),
                               torch.as_tensor(np.asarray(grad_stats.count, np.float64), device="cuda"))
    names, extras = [], []
    if adam_states:
        for name in list(cloud.param_arrays()):
            st = adam_states.get(name)
            if st is not None:
                for tag in ("m", "v"):
                    names.append((name, tag))
                    extras.append(torch.as_tensor(np.asarray(getattr(st, tag), np.float32), device="cuda"))
    out, new_stats, outs, rep = DeviceDensity().run(dev, stats, cfg, extent, rng, False, extras)
    _device_to_host_cloud(out, cloud)
    grad_stats.accum = new_stats.accum.cpu().numpy()
    grad_stats.count = new_stats.count.cpu().numpy()
    for (name, tag), t in zip(names, outs):
        setattr(adam_states[name], tag, t.cpu().numpy().astype(np.float64))
    cloud.validate()
    return {"iteration": iteration, "cloned": rep["cloned"], "split": rep["split"], "pruned": n_pruned,
            "count": rep["count"]}


def prune_only(cloud, grad_stats, cfg, adam_states=None):
    """Standalone low-opacity prune (gaussians.py:408-417); returns the number pruned."""
    dev = _host_cloud_to_device(cloud)
    stats = ViewspaceGradStats(torch.as_tensor(np.asarray(grad_stats.accum, np.float64), device="cuda"),
                               torch.as_tensor(np.asarray(grad_stats.count, np.float64), device="cuda"))
    names, extras = [], []
    if adam_states:
        for name in list(cloud.param_arrays()):
            st = adam_states.get(name)
            if st is not None:
                for tag in ("m", "v"):
                    names.append((name, tag))
                    extras.append(torch.as_tensor(np.asarray(getattr(st, tag), np.float32), device="cuda"))
    k = len(cloud)
    out, new_stats, outs, rep = DeviceDensity().run(dev, stats, cfg, 1.0, None, True, extras)
    _device_to_host_cloud(out, cloud)
    grad_stats.accum = new_stats.accum.cpu().numpy()
    grad_stats.count = new_stats.count.cpu().numpy()
    for (name, tag), t in zip(names, outs):
        setattr(adam_states[name], tag, t.cpu().numpy().astype(np.float64))
    return k - rep["count"]


def reset_opacity(cloud, cap):
    """Clamp activated opacities to at most `cap` in logit space (gaussians.py:420-425)."""
    if not 0.0 < cap < 1.0:
        raise ConfigurationError("opacity cap must lie in (0, 1)")
    if isinstance(cloud, DeviceCloud):
        t = cloud.opacity_logits
        N.check(N.load().fs4d_reset_opacity(_p(t), t.numel(), float(cap), _stream()))
        return
    t = torch.as_tensor(np.asarray(cloud.opacity_logits, np.float32), device="cuda").contiguous()
    N.check(N.load().fs4d_reset_opacity(_p(t), t.numel(), float(cap), _stream()))
    cloud.opacity_logits = t.cpu().numpy().astype(np.float64)
