"""Time-conditioned deformation on the GPU: the drop-in for
featsplat.deformation (deformation.py:19-183).

``deform`` / ``deform_with_cache`` / ``deform_backward`` keep the reference
signatures and NumPy in/out (float64 views of the fp32 device results); the
work is one fs4d_deform_fwd / fs4d_deform_bwd call each (HexPlane gather +
MLP stacks + raw-space deltas, csrc/deform.cu).  Aliasing matches the
reference: ``colors_raw`` (and ``sh_rest``) of the snapshot are the cloud's
objects, and ``features`` too when the feature branch is disabled.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, ContractViolation
from .gaussians import GaussianCloud
from .numerics import linear_layer, mlp_forward, mlp_params, set_mlp_params

BRANCHES = ("position", "rotation", "scale", "opacity")
BRANCH_DIMS = {"position": 3, "rotation": 4, "scale": 3, "opacity": 1}


@dataclass
class DeformationConfig:
    width: int = 64
    depth: int = 8
    feature_dim: int = 128
    enable_feature_update: bool = True
    enable_grid: bool = True


class DeformationNet:
    """Trunk + four extractor/head branch pairs + semantic update MLP
    (deformation.py:32-73).  Construction draws from ``rng`` in the
    reference's order so a shared seed reproduces the reference weights."""

    def __init__(self, latent_dim, cfg, rng, init="kaiming", head_init="zeros"):
        if cfg.width % 2:
            raise ConfigurationError("deformation width must be even")
        self.cfg = cfg
        self.latent_dim = latent_dim
        w, h = cfg.width, cfg.width // 2
        self.trunk = [linear_layer(latent_dim if i == 0 else w, w, "relu", rng, init)
                      for i in range(cfg.depth)]
        self.extractors, self.heads = {}, {}
        for name in BRANCHES:
            self.extractors[name] = [linear_layer(w, h, "relu", rng, init),
                                     linear_layer(h, h, "relu", rng, init)]
            self.heads[name] = [linear_layer(h, BRANCH_DIMS[name], "none", rng, head_init)]
        self.feature_mlp = [linear_layer(4 * h, h, "relu", rng, init),
                            linear_layer(h, cfg.feature_dim, "none", rng, head_init)]

    def stacks(self):
        yield "net.trunk", self.trunk
        for name in BRANCHES:
            yield f"net.ext.{name}", self.extractors[name]
            yield f"net.head.{name}", self.heads[name]
        yield "net.feat", self.feature_mlp

    def param_arrays(self):
        out = {}
        for prefix, stack in self.stacks():
            out.update(dict(mlp_params(stack, prefix)))
        return out

    def set_params(self, arrays):
        for prefix, stack in self.stacks():
            set_mlp_params(stack, prefix, arrays)


# ---------------------------------------------------------------------------
# the stacks one at a time (deformation.py:74-97), each layer on device via
# numerics.mlp_forward; deform() runs them fused on the tensor cores
# ---------------------------------------------------------------------------
def decode_hidden(net, latent):
    """Trunk output for latent [K, latent_dim]."""
    h, _ = mlp_forward(net.trunk, latent)
    return h


def decode_branches(net, hidden):
    """(deltas, feats): per branch, the head output and the extractor output."""
    deltas, feats = {}, {}
    for name in BRANCHES:
        hg, _ = mlp_forward(net.extractors[name], hidden)
        feats[name] = hg
        deltas[name], _ = mlp_forward(net.heads[name], hg)
    return deltas, feats


def update_semantics(net, branch_feats, features):
    """z' = z + F_feat([h_pos | h_rot | h_scale | h_opacity]); the features
    object itself when the update is disabled."""
    if not net.cfg.enable_feature_update:
        return features
    joint = np.concatenate([np.asarray(branch_feats[n], dtype=np.float64) for n in BRANCHES], axis=-1)
    delta, _ = mlp_forward(net.feature_mlp, joint)
    return features + delta


def _device_parts(cloud, field, net):
    from .device import DeviceCloud, DeviceField, DeviceNet
    return (DeviceCloud.from_cloud(cloud), DeviceField.from_field(field),
            DeviceNet.from_net(net))


def _engine():
    from .device import DeformEngine
    return DeformEngine()


def _host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def deform(cloud, field, net, t):
    snapshot, _ = _deform(cloud, field, net, t, False)
    return snapshot


def deform_with_cache(cloud, field, net, t):
    """Snapshot of the cloud at time t plus the backward record
    (deformation.py:105-136)."""
    return _deform(cloud, field, net, t, True)


def _deform(cloud, field, net, t, want_cache):
    if net.cfg.enable_grid and net.latent_dim != field.latent_dim:
        raise ConfigurationError(
            f"input dim {field.latent_dim} does not match first layer in_dim {net.latent_dim}")
    dc, df, dn = _device_parts(cloud, field, net)
    dcache = None
    if want_cache:
        snap, dcache = _engine().forward(dc, df, dn, t, with_cache=True)
    else:
        snap = _engine().forward(dc, df, dn, t)
    k = len(cloud)
    snapshot = GaussianCloud(
        positions=_host(snap.positions).reshape(k, 3),
        rotations=_host(snap.rotations).reshape(k, 4),
        log_scales=_host(snap.log_scales).reshape(k, 3),
        opacity_logits=_host(snap.opacity_logits).reshape(k),
        colors_raw=cloud.colors_raw,
        features=_host(snap.features).reshape(k, np.shape(cloud.features)[1])
        if net.cfg.enable_feature_update
        else cloud.features,
        sh_rest=getattr(cloud, "sh_rest", None),
    )
    cache = {"k": k, "t": float(t), "query": None if not net.cfg.enable_grid else "device",
             "feat": "device" if net.cfg.enable_feature_update else None, "device": dcache}
    return snapshot, cache


def deform_backward(cloud, field, net, cache, grads, *, deterministic=False):
    """Pull snapshot gradients back to the cloud, the net and the grid
    (deformation.py:139-183).  ``grads`` is duck-typed like the reference.
    deterministic=True (extension): fixed-point plane scatter, bitwise
    reproducible (fs4d_deform_bwd_deterministic)."""
    import torch
    from .device import DeviceCloud

    k = len(cloud)
    if cache.get("k") != k:
        raise ContractViolation("deformation cache does not match this cloud")
    dc, df, dn = _device_parts(cloud, field, net)
    d = dc.feature_dim
    f32 = dict(dtype=torch.float32, device="cuda")

    def up(name, shape):
        return torch.as_tensor(np.ascontiguousarray(getattr(grads, name), dtype=np.float32),
                               device="cuda").reshape(shape)

    feats = up("features", (k, d)) if net.cfg.enable_feature_update else torch.zeros(k, d, **f32)
    sg = DeviceCloud(up("positions", (k, 3)), up("rotations", (k, 4)), up("log_scales", (k, 3)),
                     up("opacity_logits", (k,)), torch.zeros(k, 3, **f32), feats)
    gpos, ngrads, pgrads = _engine().backward(dc, df, dn, cache["t"], sg, cache=cache.get("device"),
                                              deterministic=deterministic)

    cloud_grads = {
        "positions": _host(gpos).reshape(k, 3),
        "rotations": grads.rotations,
        "log_scales": grads.log_scales,
        "opacity_logits": grads.opacity_logits,
        "features": grads.features,
    }
    if not net.cfg.enable_grid:
        cloud_grads["positions"] = np.array(grads.positions, dtype=np.float64, copy=True)
    net_grads = {}
    for prefix, stack in ngrads.layers.items():
        if prefix == "net.feat" and not net.cfg.enable_feature_update:
            continue
        for i, (w, b, _) in enumerate(stack):
            net_grads[f"{prefix}.{i}.weight"] = _host(w)
            net_grads[f"{prefix}.{i}.bias"] = _host(b)
    plane_grads = None
    if pgrads is not None:
        plane_grads = [[_host(p) for p in level] for level in pgrads.planes]
    return cloud_grads, net_grads, plane_grads
