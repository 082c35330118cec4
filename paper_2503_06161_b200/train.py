"""Data-parallel training step of the render path on device (configs[4], and
the reference's fine-stage iteration training.py:489-535 when the decoder /
TV / optimizer options are on).

Per rank: a batch of (view, t) pairs; for each pair
    fs4d_deform_fwd -> fs4d_render_fwd -> loss + upstream image gradients
    -> fs4d_render_bwd -> fs4d_deform_bwd (accumulating into the flat buffer)
then the HexPlane TV term (hexplane.py:190-222) is folded into the plane
gradients, ONE all-reduce (SUM) of the flat gradient buffer runs, and --
with an optimizer attached -- one multi-segment Adam launch
(numerics.py:137-159) updates every parameter array with its own schedule
(training.py:156-170, 365-376, 431-442).  The mean over pairs and ranks is
folded into the loss weights, so the collective is a plain SUM.

Loss modes:
  "raw"     configs[4]: L1 RGB / (3HW) + L1 raw D-channel feature / (HW) at
            render resolution (fused kernel fs4d_l1_loss_grad).
  "decoder" the reference's fine stage: masked photometric L1 (+ depth L1)
            (training.py:300-338) and the pointwise-decoder feature loss
            against a teacher map (training.py:497-505) in one fused kernel.
"""

import collections
import ctypes
import os

import numpy as np
import torch

from . import _native as N
from .device import (DeformEngine, DeviceCloud, DeviceField, DeviceNet, Renderer, StatusBlock, _p, _stream,
                     locality_order)
from .errors import NumericalError
from .hexplane import tv_loss_grad_device
from .numerics import lr_at_step
from .optim import FlatAdam
from .parallel import FlatGrads, gradient_specs
from .semantic import DecoderLoss


def photometric_loss_grad(color, image, mask, depth, depth_target, alpha, lambda_rgb, lambda_depth, d_color,
                          d_depth=None, terms=None, loss=None, workspace=None):
    """Masked photometric L1 + depth L1 and their gradients (training.py:300-338)
    on device.  Returns the device float64 terms tensor {rgb, depth, n_rgb, n_d}."""
    lib = N.load()
    h, w = int(color.shape[0]), int(color.shape[1])
    if terms is None:
        terms = torch.zeros(4, dtype=torch.float64, device=color.device)
    need = int(lib.fs4d_photometric_workspace_bytes(h, w))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=color.device)
    N.check(lib.fs4d_photometric_loss_grad(_p(color), _p(image), _p(mask), _p(depth), _p(depth_target), _p(alpha),
                                           h, w, float(lambda_rgb), float(lambda_depth), _p(d_color), _p(d_depth),
                                           _p(terms), _p(loss), _p(workspace), workspace.numel(), _stream()))
    return terms


def _net_layer_specs(net):
    specs = []
    for prefix, stack in net.layers.items():
        for i, (wt, b, _) in enumerate(stack):
            specs += [(f"{prefix}.{i}.weight", tuple(wt.shape)), (f"{prefix}.{i}.bias", tuple(b.shape))]
    return specs


class TrainStep:
    def __init__(self, cloud, field, net, height, width, cfg, world=1, group=None, device="cuda",
                 loss_mode="raw", lambda_rgb=1.0, lambda_depth=0.0, lambda_feat=1.0, lambda_tv=0.0,
                 decoder=None, locality=None, lanes=None, deterministic=False):
        self.cloud, self.field, self.net = cloud, field, net
        self.h, self.w, self.cfg = int(height), int(width), cfg
        self.world, self.group = int(world), group
        self.device = device
        if loss_mode not in ("raw", "decoder"):
            raise ValueError(f"unknown loss mode {loss_mode!r}")
        self.loss_mode = loss_mode
        # bitwise reproducible steps: ordered blend-backward partials, fixed-
        # point plane scatter, one loss scalar per lane summed in lane order
        # (the reference's resume test, test_training.py:282-299)
        self.deterministic = bool(deterministic)
        self.locality = (os.environ.get("FS4D_TRAIN_LOCALITY", "0") == "1") if locality is None else bool(locality)
        # pairs in flight: lane j runs pairs j, j+L, ... on its own stream with
        # its own snapshot / record / image gradients / gradient buffer; the
        # lane buffers are summed into self.grads before the all-reduce
        self.n_lanes = max(1, int(os.environ.get("FS4D_TRAIN_LANES", "3") if lanes is None else lanes))
        self._lanes = None
        # two-bucket gradient exchange overlapping the backward: always at
        # world > 1; FS4D_OVERLAP_ALLREDUCE=1 also takes that path at world 1
        self.overlap_allreduce = os.environ.get("FS4D_OVERLAP_ALLREDUCE", "0") == "1"
        self._comm_stream = None
        self.lambda_rgb, self.lambda_depth = float(lambda_rgb), float(lambda_depth)
        self.lambda_feat, self.lambda_tv = float(lambda_feat), float(lambda_tv)
        self.decoder = decoder  # (weight [Ct,N], bias [Ct]) CUDA tensors for loss_mode="decoder"
        self.deformer = DeformEngine(device)
        self.renderer = Renderer(device)
        k, d, sh = len(cloud), cloud.feature_dim, cloud.sh_degree
        plane_shapes = [[tuple(p.shape) for p in level] for level in field.planes]
        specs = gradient_specs(k, d, sh, plane_shapes, _net_layer_specs(net))
        if decoder is not None:
            specs += [("decoder.weight", tuple(decoder[0].shape)), ("decoder.bias", tuple(decoder[1].shape))]
        self.specs = specs
        self.grads = FlatGrads(specs, device)
        self.cloud_grads, self.plane_grads, self.net_grads = self._bind(self.grads)
        self.snap = DeviceCloud.empty(k, d, 0, device)
        self.snap_grads = DeviceCloud.empty(k, d, sh, device)
        dout = d if cfg.with_features else 0
        self.images = self.renderer.alloc_images(self.h, self.w, dout)
        f = dict(dtype=torch.float32, device=device)
        self.d_color = torch.empty(self.h, self.w, 3, **f)
        self.d_depth = torch.empty(self.h, self.w, **f)
        self.d_feature = torch.empty(self.h, self.w, dout, **f)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.cache = None  # deform_with_cache activations, reused pair to pair
        self.decoder_loss = DecoderLoss(device)
        self.photo_ws = None
        self.params = None
        self.optimizer = None
        self.schedules = None
        self.iteration = 0
        self.stats = None      # ViewspaceGradStats on device when track_stats() is on
        self.vs_norm = None
        # asynchronous error reporting: every step copies its status blocks
        # (one per lane + the Adam block) to pinned host memory; the next
        # run() (or sync()) inspects them and raises
        self._pending = collections.deque()

    def _bind(self, flat):
        """DeviceCloud / DeviceField / DeviceNet views into a flat buffer."""
        g = flat
        cloud = DeviceCloud(g["positions"], g["rotations"], g["log_scales"], g["opacity_logits"], g["colors_raw"],
                            g["features"], g.views.get("sh_rest"))
        planes = DeviceField([[g[f"grid.l{l}.p{p}"] for p in range(len(level))]
                              for l, level in enumerate(self.field.planes)], self.field.aabb, self.field.channels)
        net = DeviceNet({prefix: [(g[f"{prefix}.{i}.weight"], g[f"{prefix}.{i}.bias"], relu)
                                  for i, (_, _, relu) in enumerate(stack)]
                         for prefix, stack in self.net.layers.items()},
                        self.net.latent_dim, self.net.width, self.net.depth, self.net.feature_dim,
                        self.net.enable_grid, self.net.enable_feature_update)
        return cloud, planes, net

    def attach_optimizer(self, schedules):
        """Move every parameter into ONE flat fp32 buffer (same layout as the
        gradients) and attach a multi-segment Adam.  schedules: schedule key
        (positions, rotations, log_scales, opacity_logits, colors_raw,
        features, grid, net, decoder -- TrainConfig.schedules(),
        training.py:156-170) -> numerics.LrSchedule.  sh_rest uses the
        colors_raw schedule."""
        params = FlatGrads(self.specs, self.device)
        cloud, field, net = self._bind(params)
        for name in DeviceCloud.FIELDS + ("sh_rest",):
            src = getattr(self.cloud, name)
            if src is not None and getattr(cloud, name) is not None:
                getattr(cloud, name).copy_(src)
        for l, level in enumerate(self.field.planes):
            for p, plane in enumerate(level):
                field.planes[l][p].copy_(plane)
        for prefix, stack in self.net.layers.items():
            for i, (wt, b, _) in enumerate(stack):
                net.layers[prefix][i][0].copy_(wt)
                net.layers[prefix][i][1].copy_(b)
        if self.decoder is not None:
            params["decoder.weight"].copy_(self.decoder[0])
            params["decoder.bias"].copy_(self.decoder[1])
            self.decoder = (params["decoder.weight"], params["decoder.bias"])
        self.cloud, self.field, self.net = cloud, field, net
        self.params = params
        self.schedules = dict(schedules)
        self.schedules.setdefault("sh_rest", self.schedules.get("colors_raw"))
        self.optimizer = FlatAdam(self.specs, params.buffer, offsets=params.offsets)
        return self

    def current_lrs(self):
        return {k: lr_at_step(s, self.iteration) for k, s in self.schedules.items() if s is not None}

    def _make_lanes(self):
        from types import SimpleNamespace
        k, d, sh = len(self.cloud), self.cloud.feature_dim, self.cloud.sh_degree
        dout = self.d_feature.shape[2]
        f = dict(dtype=torch.float32, device=self.device)
        lanes = []
        for j in range(self.n_lanes):
            if j == 0:
                ln = SimpleNamespace(grads=self.grads, cloud_grads=self.cloud_grads, plane_grads=self.plane_grads,
                                     net_grads=self.net_grads, deformer=self.deformer, renderer=self.renderer,
                                     snap=self.snap, snap_grads=self.snap_grads, images=self.images,
                                     d_color=self.d_color, d_depth=self.d_depth, d_feature=self.d_feature,
                                     decoder_loss=self.decoder_loss, vs_norm=self.vs_norm)
            else:
                g = FlatGrads(self.specs, self.device)
                cg, pg, ng = self._bind(g)
                ln = SimpleNamespace(grads=g, cloud_grads=cg, plane_grads=pg, net_grads=ng,
                                     deformer=DeformEngine(self.device), renderer=Renderer(self.device),
                                     snap=DeviceCloud.empty(k, d, 0, self.device),
                                     snap_grads=DeviceCloud.empty(k, d, sh, self.device),
                                     images=self.renderer.alloc_images(self.h, self.w, dout),
                                     d_color=torch.empty(self.h, self.w, 3, **f), d_depth=torch.empty(self.h, self.w, **f),
                                     d_feature=torch.empty(self.h, self.w, dout, **f),
                                     decoder_loss=DecoderLoss(self.device),
                                     vs_norm=None if self.vs_norm is None else torch.empty_like(self.vs_norm))
            ln.cache, ln.photo_ws = None, None
            ln.step_status = StatusBlock(self.device)  # every render of this lane's pairs, merged
            ln.loss = torch.zeros(1, dtype=torch.float64, device=self.device) if self.deterministic else self.loss
            ln.stream = torch.cuda.Stream(device=self.device) if self.n_lanes > 1 else None
            lanes.append(ln)
        self._lanes = lanes
        return lanes

    @property
    def _early_span(self):
        """Flat-buffer range of the pass-through cloud gradients (rotations ..
        features): final after each lane's last pass-through kernel."""
        return self.grads.span("rotations", "features")

    def active_arrays(self, batch):
        """Parameter arrays that receive a gradient this iteration -- the keys
        of the reference's `grads` dict (training.py:509-531): `features`
        only with feature supervision, grid.* only with the HexPlane,
        net.feat.* only with the feature update, decoder.* only when the
        decoder loss ran.  The others are left out of the Adam step."""
        dout = self.d_feature.shape[2]
        if self.loss_mode == "raw":
            feature_on = dout > 0
        else:
            feature_on = dout > 0 and self.decoder is not None and any(
                len(it) > 4 and it[4] is not None for it in batch)
        act = set()
        for name, _ in self.specs:
            if name == "features" and not feature_on:
                continue
            if name.startswith("grid.") and not self.net.enable_grid:
                continue
            if name.startswith("net.feat.") and not self.net.enable_feature_update:
                continue
            if name.startswith("decoder.") and not feature_on:
                continue
            act.add(name)
        return act

    def run(self, batch, check=False):
        """batch: list of (t, K, T, target_rgb [H,W,3], target_feat) CUDA
        tensors; loss_mode "decoder" additionally takes optional
        (mask uint8 [H,W] | None, target_depth [H,W] | None) as items 5-6 and
        target_feat is the teacher map [ho,wo,Ct].  Returns the device loss
        (mean over pairs and ranks after the reduce).

        check=False keeps the step asynchronous: device errors of THIS step
        (tile-pair overflow, non-finite snapshot or gradient) skip its Adam
        update on the device and are raised by the next run() or sync()."""
        self._poll(block=False)
        lib = N.load()
        n = len(batch) * self.world
        w = 1.0 / n
        self.loss.zero_()
        dout = self.d_feature.shape[2]
        field = self.field
        if self.locality:
            # Morton visiting order of this step's canonical positions for the
            # HexPlane gather / scatter (identical results, coherent caches)
            field = field.with_order(locality_order(self.cloud.positions, field.aabb, self.device))
        lanes = self._lanes or self._make_lanes()
        nl = len(lanes)
        main = torch.cuda.current_stream()
        for ln in lanes:
            ln.step_status.reset()
            if self.deterministic:
                ln.loss.zero_()
        if nl > 1:
            ready = torch.cuda.Event()
            ready.record(main)
            for ln in lanes:
                ln.stream.wait_event(ready)
        stats_done = None  # the stats accumulation is a plain += : serialised across lanes
        used = lanes[:min(nl, len(batch))]
        # gradient exchange in two buckets: the pass-through
        # cloud rows (rotations .. features, ~80% of the buffer) are final once
        # every lane's LAST pair has run its pass-through kernel, so their lane
        # sum + all-reduce run on a side stream while those pairs' MLP and
        # HexPlane backward still run; positions, planes, MLP and decoder
        # follow after the backward.  Same sums in the same order: results are
        # identical to one all-reduce of the whole buffer.
        overlap = self.world > 1 or self.overlap_allreduce
        last_pair = {i % nl: i for i in range(len(batch))}
        pass_events = {}
        for i, item in enumerate(batch):
            ln = lanes[i % nl]
            first = i < nl
            ev = None
            if overlap and last_pair[i % nl] == i:
                ev = pass_events[i % nl] = torch.cuda.Event()
            with torch.cuda.stream(ln.stream if nl > 1 else main):
                stats_done = self._run_pair(ln, item, field, w, dout, first, check, stats_done, pass_event=ev)
        lo, hi = self._early_span if overlap else (0, 0)

        def lane_sum(a, b):  # lane 0's buffer[a:b] += the other lanes', one pass
            if len(used) > 1 and b > a:
                srcs = (ctypes.c_void_p * (len(used) - 1))(*[ln.grads.buffer.data_ptr() + 4 * a for ln in used[1:]])
                N.check(lib.fs4d_sum_buffers(self.grads.buffer.data_ptr() + 4 * a, srcs, len(used) - 1, b - a, 1,
                                             _stream()))
        early = None
        if overlap:
            if self._comm_stream is None:
                self._comm_stream = torch.cuda.Stream(device=self.device)
            comm = self._comm_stream
            comm.wait_stream(main)  # buffers of the previous step
            for ev in pass_events.values():
                comm.wait_event(ev)
            with torch.cuda.stream(comm):
                lane_sum(lo, hi)
                early = self.grads.allreduce_sum_range(lo, hi, self.group, async_op=True)
        if nl > 1:
            for ln in used:
                main.wait_stream(ln.stream)
            lane_sum(0, lo)
            lane_sum(hi, self.grads.numel)
        if self.deterministic:
            for ln in used:  # the lanes' losses in lane order
                self.loss.add_(ln.loss)
        if self.lambda_tv > 0 and self.net.enable_grid:
            # d(lambda_tv * tv)/d(plane) once per iteration (training.py:523-529); 1/world per rank
            tv_loss_grad_device(self.field, self.plane_grads, self.lambda_tv / self.world, True, self.loss)
        if overlap:
            self.grads.allreduce_sum_range(0, lo, self.group)
            self.grads.allreduce_sum_range(hi, self.grads.numel, self.group)
            if early is not None:
                early.wait()  # the current (main) stream waits for the early bucket
            main.wait_stream(self._comm_stream)
        else:
            self.grads.allreduce_sum(self.group)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.loss, op=dist.ReduceOp.SUM, group=self.group)
        if self.optimizer is not None:
            self.optimizer.step(self.grads.buffer, self.current_lrs(), active=self.active_arrays(batch),
                                guards=[ln.step_status.t for ln in used])
            self.iteration += 1
        self._post_status(used)
        if check:
            self.sync()
        return self.loss

    _MAX_PENDING = 2  # steps whose status may still be in flight before run() blocks on the oldest

    def _post_status(self, used):
        """Queue the D2H copy of this step's status blocks (pinned, async)."""
        rows = len(used) + 1
        host = torch.zeros((rows, N.STATUS_WORDS), dtype=torch.int32).pin_memory()
        for j, ln in enumerate(used):
            host[j].copy_(ln.step_status.t, non_blocking=True)
        if self.optimizer is not None:
            host[len(used)].copy_(self.optimizer.status.t, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._pending.append((ev, list(used), self.optimizer is not None, host))

    def _poll(self, block):
        """Inspect finished steps' status copies in order (all of them when
        `block`, else the completed ones plus enough to keep at most
        _MAX_PENDING in flight)."""
        while self._pending:
            ev = self._pending[0][0]
            if not (block or ev.query() or len(self._pending) > self._MAX_PENDING):
                break
            ev.synchronize()
            self._inspect(*self._pending.popleft()[1:])

    def sync(self):
        """Wait for every queued step's status and raise its device error,
        if any: a tile-pair overflow grows that lane's pair buffer first (so
        re-running the batch succeeds) and raises CapacityError; a
        non-finite snapshot or gradient raises NumericalError.  Either way
        that step's Adam update was skipped on the device, so its parameters,
        moments and step counts stayed as they were and `iteration` is
        rolled back by one."""
        self._poll(block=True)

    def _inspect(self, used, has_opt, host):
        st = host.numpy()
        failed = None
        for j, ln in enumerate(used):
            row = st[j]
            code = int(row[N.ST_CODE])
            if code == N.ERR_CAPACITY:
                pairs = (int(row[N.ST_PAIRS_HI]) << 32) | (int(row[N.ST_PAIRS_LO]) & 0xFFFFFFFF)
                ln.renderer.cap = max(int(ln.renderer.cap or 0), int(pairs * 1.25) + 1024)
            if code != N.OK and failed is None:
                failed = row.copy()
        if has_opt and failed is None and int(st[len(used)][N.ST_CODE]) != N.OK:
            failed = st[len(used)].copy()
        if failed is None:
            return
        self._pending.clear()
        if has_opt:
            self.iteration -= 1
            seg = int(failed[N.ST_ADAM_BAD_SEG])
            if int(failed[N.ST_CODE]) == N.ERR_NUMERIC and seg not in (N.ADAM_GATED, 0x7FFFFFFF):
                self.optimizer.check(failed)  # non-finite gradient: names the parameter array
        try:
            N.raise_device_status(failed)
        except Exception as e:
            raise type(e)(f"training step skipped on the device (parameters unchanged): {e}") from None

    def _run_pair(self, ln, item, field, w, dout, first, check, stats_done, pass_event=None):
        """One (view, t) pair on lane `ln` (the current stream): deform, render,
        loss + image gradients, render backward, deform backward into the
        lane's gradient buffer (overwritten by the lane's first pair)."""
        lib = N.load()
        t, K, T, tgt_rgb, tgt_feat = item[:5]
        _, ln.cache = ln.deformer.forward(self.cloud, field, self.net, t, out=ln.snap, with_cache=ln.cache or True)
        imgs, rec = ln.renderer.forward(ln.snap, K, T, self.h, self.w, self.cfg, images=ln.images, check=check)
        N.check(lib.fs4d_status_merge(_p(ln.renderer.status.t), _p(ln.step_status.t), 0, _stream()))
        d_depth = None
        if self.loss_mode == "raw":
            N.check(lib.fs4d_l1_loss_grad(_p(imgs["color"]), _p(tgt_rgb), _p(imgs["feature"]) if dout else None,
                                          _p(tgt_feat) if dout else None, self.h, self.w, dout,
                                          w * self.lambda_rgb, w * self.lambda_feat, _p(ln.d_color),
                                          _p(ln.d_feature) if dout else None, _p(ln.loss), _stream()))
        else:
            mask = item[5] if len(item) > 5 else None
            tgt_depth = item[6] if len(item) > 6 else None
            if tgt_depth is not None:
                d_depth = ln.d_depth
            if ln.photo_ws is None:
                ln.photo_ws = torch.empty(int(lib.fs4d_photometric_workspace_bytes(self.h, self.w)),
                                          dtype=torch.uint8, device=self.device)
            photometric_loss_grad(imgs["color"], tgt_rgb, mask, imgs["depth"] if d_depth is not None else None,
                                  tgt_depth, imgs["alpha"], w * self.lambda_rgb, w * self.lambda_depth,
                                  ln.d_color, d_depth, loss=ln.loss, workspace=ln.photo_ws)
            if dout and tgt_feat is not None and self.decoder is not None:
                ln.decoder_loss(self.decoder[0], self.decoder[1], imgs["feature"], tgt_feat, w * self.lambda_feat,
                                ln.d_feature, ln.grads["decoder.weight"], ln.grads["decoder.bias"], ln.loss,
                                accumulate=not first)
            elif dout:
                ln.d_feature.zero_()
        ln.renderer.backward(ln.snap, K, T, self.h, self.w, self.cfg, rec, d_color=ln.d_color, d_depth=d_depth,
                             d_feature=ln.d_feature if dout else None, grads=ln.snap_grads,
                             viewspace=ln.vs_norm if self.stats is not None else False,
                             deterministic=self.deterministic)
        if self.stats is not None:  # training.py:514 grad_stats.add (dense, source order)
            cur = torch.cuda.current_stream()
            if stats_done is not None:
                cur.wait_event(stats_done)
            self.stats.add_dense(ln.vs_norm)
            stats_done = torch.cuda.Event()
            stats_done.record(cur)
        ln.deformer.backward(self.cloud, field, self.net, t, ln.snap_grads, cloud_grads=ln.cloud_grads,
                             net_grads=ln.net_grads, plane_grads=ln.plane_grads if self.net.enable_grid else None,
                             accumulate=not first, cache=ln.cache, deterministic=self.deterministic,
                             pass_event=pass_event)
        return stats_done

    # ------------------------------------------------------------------
    # adaptive density control in the training loop (training.py:445-456)
    # ------------------------------------------------------------------
    def track_stats(self):
        """Accumulate the view-space gradient statistics every step
        (ViewspaceGradStats on device, reset by densify)."""
        from .density import ViewspaceGradStats
        k = len(self.cloud)
        self.stats = ViewspaceGradStats.zeros(k, self.device)
        self.vs_norm = torch.empty(max(k, 1), dtype=torch.float32, device=self.device)
        self._lanes = None
        return self

    def densify(self, cfg, extent, rng, prune_only=False):
        """densify_and_prune / prune_only (gaussians.py:349-417) on the device
        parameters: compacts every per-Gaussian parameter array and its Adam
        moments in the reference's row order, keeps the network / plane /
        decoder parameters, moments and every step count, rebuilds the flat
        parameter / gradient / moment buffers for the new K and resets the
        statistics.  Returns the reference's report dict."""
        from .density import DeviceDensity, ViewspaceGradStats
        from .parallel import PER_GAUSSIAN
        if self.optimizer is None:
            raise ValueError("attach_optimizer() first: density control remaps the Adam moments")
        per = [n for n, _ in PER_GAUSSIAN if n in self.params.views]
        old_specs, old_params, old_opt = self.specs, self.params, self.optimizer
        extras = []
        for n in per:
            i = [sn for sn, _ in old_specs].index(n)
            off, cnt = old_params.offsets[i], old_params.sizes[i]
            shape = old_params.views[n].shape
            extras += [old_opt.m[off:off + cnt].view(shape), old_opt.v[off:off + cnt].view(shape)]
        self.sync()
        stats = self.stats if self.stats is not None else ViewspaceGradStats.zeros(len(self.cloud), self.device)
        if self.world > 1:
            # every rank saw different (view, t) pairs: classify on the sums
            # over all ranks, as a single process training on the union would
            # (SURVEY §8(e)); the split samples must come from the same seeded
            # rng on every rank (gaussians.py:380-383)
            import torch.distributed as dist
            dist.all_reduce(stats.accum, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(stats.count, op=dist.ReduceOp.SUM, group=self.group)
        out, new_stats, outs, rep = DeviceDensity(self.device).run(self.cloud, stats, cfg, extent, rng, prune_only,
                                                                   extras)
        k = len(out)
        if self.world > 1:
            import torch.distributed as dist
            ks = torch.tensor([k, -k], dtype=torch.int64, device=self.device)
            dist.all_reduce(ks, op=dist.ReduceOp.MAX, group=self.group)
            if int(ks[0]) != k or -int(ks[1]) != k:
                raise RuntimeError(f"density control diverged across ranks (K = {k} here, range "
                                   f"[{-int(ks[1])}, {int(ks[0])}]): seed the split rng identically on every rank")
        d, sh = out.feature_dim, out.sh_degree
        field_specs = [(n, sh_) for n, sh_ in old_specs if n not in per]
        new_specs = gradient_specs(k, d, sh, [], []) + field_specs
        params = FlatGrads(new_specs, self.device)
        opt = FlatAdam(new_specs, params.buffer, offsets=params.offsets)
        moved = dict(zip([(n, t) for n in per for t in ("m", "v")], outs))
        for i, (n, _) in enumerate(new_specs):
            off, cnt = params.offsets[i], params.sizes[i]
            if n in per:
                src = getattr(out, n)
                params.buffer[off:off + cnt].copy_(src.reshape(-1))
                opt.m[off:off + cnt].copy_(moved[(n, "m")].reshape(-1))
                opt.v[off:off + cnt].copy_(moved[(n, "v")].reshape(-1))
            else:
                j = [sn for sn, _ in old_specs].index(n)
                o2, c2 = old_params.offsets[j], old_params.sizes[j]
                params.buffer[off:off + cnt].copy_(old_params.buffer[o2:o2 + c2])
                opt.m[off:off + cnt].copy_(old_opt.m[o2:o2 + c2])
                opt.v[off:off + cnt].copy_(old_opt.v[o2:o2 + c2])
        # step counts follow their arrays (AdamState per array, numerics.py:122-133)
        old_steps = old_opt.steps.cpu().tolist()
        name_to_step = {n: old_steps[i] for i, (n, _) in enumerate(old_specs)}
        opt.steps.copy_(torch.tensor([name_to_step[n] for n, _ in new_specs], dtype=torch.int32))
        self.specs, self.params, self.optimizer = new_specs, params, opt
        self.cloud, self.field, self.net = self._bind(params)
        if self.decoder is not None:
            self.decoder = (params["decoder.weight"], params["decoder.bias"])
        self.grads = FlatGrads(new_specs, self.device)
        self.cloud_grads, self.plane_grads, self.net_grads = self._bind(self.grads)
        self.snap = DeviceCloud.empty(k, d, 0, self.device)
        self.snap_grads = DeviceCloud.empty(k, d, sh, self.device)
        self.cache = None
        self._lanes = None
        if self.stats is not None:
            self.stats = new_stats  # reset (densify) or compacted (prune_only), gaussians.py:397-415
            self.vs_norm = torch.empty(max(k, 1), dtype=torch.float32, device=self.device)
        return rep
