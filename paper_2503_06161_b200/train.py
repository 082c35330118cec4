"""Data-parallel training step of the render path on device (configs[4]).

Per rank: a batch of (view, t) pairs; for each pair
    fs4d_deform_fwd -> fs4d_render_fwd -> fs4d_l1_loss_grad (L1 RGB + L1
    feature, training.py:302-338 / semantic.py:171-181 normalisations)
    -> fs4d_render_bwd -> fs4d_deform_bwd (accumulating into the flat buffer)
then ONE all-reduce (SUM) of the flat gradient buffer; the mean over pairs
and ranks is folded into the loss weights.  The optimizer step is the next
row; this module stops at the reduced gradients.
"""

import ctypes

import torch

from . import _native as N
from .device import DeformEngine, DeviceCloud, DeviceField, DeviceNet, Renderer, _p, _stream
from .parallel import FlatGrads, gradient_specs


class TrainStep:
    def __init__(self, cloud, field, net, height, width, cfg, world=1, group=None, device="cuda"):
        self.cloud, self.field, self.net = cloud, field, net
        self.h, self.w, self.cfg = int(height), int(width), cfg
        self.world, self.group = int(world), group
        self.deformer = DeformEngine(device)
        self.renderer = Renderer(device)
        k, d, sh = len(cloud), cloud.feature_dim, cloud.sh_degree
        layer_shapes = []
        for prefix, stack in net.layers.items():
            for i, (wt, b, _) in enumerate(stack):
                layer_shapes += [(f"{prefix}.{i}.weight", tuple(wt.shape)), (f"{prefix}.{i}.bias", tuple(b.shape))]
        plane_shapes = [[tuple(p.shape) for p in level] for level in field.planes]
        self.grads = FlatGrads(gradient_specs(k, d, sh, plane_shapes, layer_shapes), device)
        g = self.grads
        self.cloud_grads = DeviceCloud(g["positions"], g["rotations"], g["log_scales"], g["opacity_logits"],
                                       g["colors_raw"], g["features"], g.views.get("sh_rest"))
        self.plane_grads = DeviceField([[g[f"grid.l{l}.p{p}"] for p in range(len(level))]
                                        for l, level in enumerate(field.planes)], field.aabb, field.channels)
        self.net_grads = DeviceNet({prefix: [(g[f"{prefix}.{i}.weight"], g[f"{prefix}.{i}.bias"], relu)
                                             for i, (_, _, relu) in enumerate(stack)]
                                    for prefix, stack in net.layers.items()},
                                   net.latent_dim, net.width, net.depth, net.feature_dim, net.enable_grid,
                                   net.enable_feature_update)
        self.snap = DeviceCloud.empty(k, d, 0, device)
        self.snap_grads = DeviceCloud.empty(k, d, sh, device)
        dout = d if cfg.with_features else 0
        self.images = self.renderer.alloc_images(self.h, self.w, dout)
        f = dict(dtype=torch.float32, device=device)
        self.d_color = torch.empty(self.h, self.w, 3, **f)
        self.d_feature = torch.empty(self.h, self.w, dout, **f)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.cache = None  # deform_with_cache activations, reused pair to pair

    def run(self, batch, check=False):
        """batch: list of (t, K, T, target_rgb [H,W,3] cuda, target_feat [H,W,D] cuda).
        Returns the device loss (mean over pairs and ranks after the reduce)."""
        lib = N.load()
        n = len(batch) * self.world
        w = 1.0 / n
        self.loss.zero_()
        dout = self.d_feature.shape[2]
        for i, (t, K, T, tgt_rgb, tgt_feat) in enumerate(batch):
            _, self.cache = self.deformer.forward(self.cloud, self.field, self.net, t, out=self.snap,
                                                  with_cache=self.cache or True)
            imgs, rec = self.renderer.forward(self.snap, K, T, self.h, self.w, self.cfg, images=self.images,
                                              check=check)
            N.check(lib.fs4d_l1_loss_grad(_p(imgs["color"]), _p(tgt_rgb), _p(imgs["feature"]) if dout else None,
                                          _p(tgt_feat) if dout else None, self.h, self.w, dout, w, w,
                                          _p(self.d_color), _p(self.d_feature) if dout else None,
                                          _p(self.loss), _stream()))
            self.renderer.backward(self.snap, K, T, self.h, self.w, self.cfg, rec, d_color=self.d_color,
                                   d_feature=self.d_feature if dout else None, grads=self.snap_grads)
            self.deformer.backward(self.cloud, self.field, self.net, t, self.snap_grads,
                                   cloud_grads=self.cloud_grads, net_grads=self.net_grads,
                                   plane_grads=self.plane_grads if self.net.enable_grid else None,
                                   accumulate=i > 0, cache=self.cache)
        self.grads.allreduce_sum(self.group)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.loss, op=dist.ReduceOp.SUM, group=self.group)
        return self.loss
