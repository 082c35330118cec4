"""Device-resident (torch CUDA) fast path over libfs4d.

PyTorch is only the allocator/stream provider here: every op is one call into
the C ABI (include/fs4d.h) on the current CUDA stream.  Objects:

  DeviceCloud   GaussianCloud as fp32 SoA tensors (gaussians.py:39-94)
  DeviceField   HexPlaneField planes + aabb (hexplane.py:49-92)
  DeviceNet     DeformationNet weights (deformation.py:32-73)
  Renderer      owns the render record (workspace) + status block and grows
                the tile-pair capacity on overflow (no host sync in steady
                state when check=False)

The numpy-facing modules (rasterizer, deformation) wrap these to keep the
reference API unchanged.
"""

import ctypes
import os

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, ContractViolation

BRANCHES = ("position", "rotation", "scale", "opacity")
BRANCH_DIMS = (3, 4, 3, 1)


def _p(t):
    """Device address of a tensor (None -> NULL), usable as a ctypes c_void_p
    argument or struct field."""
    return None if t is None else t.data_ptr()


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(x, device):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=device)


class DeviceCloud:
    """fp32 SoA cloud on the GPU. sh_rest is [K, (L+1)^2 - 1, 3] or None."""

    FIELDS = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features")

    def __init__(self, positions, rotations, log_scales, opacity_logits, colors_raw, features,
                 sh_rest=None):
        self.positions = positions
        self.rotations = rotations
        self.log_scales = log_scales
        self.opacity_logits = opacity_logits
        self.colors_raw = colors_raw
        self.features = features
        self.sh_rest = sh_rest

    def __len__(self):
        return self.positions.shape[0]

    @property
    def feature_dim(self):
        return self.features.shape[1]

    @property
    def sh_degree(self):
        if self.sh_rest is None or self.sh_rest.shape[1] == 0:
            return 0
        return int(round(np.sqrt(self.sh_rest.shape[1] + 1))) - 1

    @classmethod
    def from_cloud(cls, cloud, device="cuda"):
        sh = getattr(cloud, "sh_rest", None)
        k = len(cloud)
        d = int(np.shape(cloud.features)[1]) if np.ndim(cloud.features) == 2 else 0
        return cls(_dev(cloud.positions, device).reshape(k, 3),
                   _dev(cloud.rotations, device).reshape(k, 4),
                   _dev(cloud.log_scales, device).reshape(k, 3),
                   _dev(cloud.opacity_logits, device).reshape(k),
                   _dev(cloud.colors_raw, device).reshape(k, 3),
                   _dev(cloud.features, device).reshape(k, d),
                   None if sh is None else _dev(sh, device).reshape(k, np.shape(sh)[1], 3))

    @classmethod
    def empty(cls, k, d, sh_degree=0, device="cuda"):
        f = dict(dtype=torch.float32, device=device)
        n_sh = (sh_degree + 1) ** 2 - 1
        return cls(torch.empty(k, 3, **f), torch.empty(k, 4, **f), torch.empty(k, 3, **f),
                   torch.empty(k, **f), torch.empty(k, 3, **f), torch.empty(k, d, **f),
                   torch.empty(k, n_sh, 3, **f) if n_sh > 0 else None)

    def struct(self):
        s = N.Cloud()
        s.K = len(self)
        s.D = self.feature_dim
        s.sh_degree = self.sh_degree
        for name in self.FIELDS:
            setattr(s, name, _p(getattr(self, name)))
        s.sh_rest = _p(self.sh_rest)
        return s


def camera_struct(K, T, height, width):
    c = N.Camera()
    c.height = int(height)
    c.width = int(width)
    c.K[:] = [float(v) for v in np.asarray(K, dtype=np.float64).reshape(9)]
    c.T[:] = [float(v) for v in np.asarray(T, dtype=np.float64).reshape(16)]
    return c


def raster_struct(cfg):
    r = N.RasterCfg()
    r.tile = int(cfg.tile)
    r.with_features = int(bool(cfg.with_features))
    r.z_near = float(cfg.z_near)
    r.lowpass = float(cfg.lowpass)
    r.alpha_cap = float(cfg.alpha_cap)
    r.alpha_skip = float(cfg.alpha_skip)
    r.stop_transmittance = float(cfg.stop_transmittance)
    bg = np.zeros(3) if cfg.background is None else np.asarray(cfg.background, dtype=np.float64)
    r.background[:] = [float(v) for v in bg.reshape(3)]
    return r


class StatusBlock:
    """Device int32[32] status words (FS4D_ST_*), reset before each call."""

    def __init__(self, device="cuda"):
        self.t = torch.zeros(N.STATUS_WORDS, dtype=torch.int32, device=device)

    def reset(self):
        N.check(N.load().fs4d_status_reset(_p(self.t), _stream()))

    def read(self):
        return self.t.cpu().numpy()

    def raise_if_error(self):
        st = self.read()
        N.raise_device_status(st)
        return st


class DeviceField:
    """HexPlane planes [levels][6] of [Ra, Rb, C] fp32 plus the aabb."""

    def __init__(self, planes, aabb, channels, order=None):
        self.planes = planes
        self.aabb = np.asarray(aabb, dtype=np.float64).reshape(2, 3)
        self.channels = int(channels)
        self.order = order  # optional int32 [K] Gaussian visiting order (locality_order)

    @property
    def levels(self):
        return len(self.planes)

    @property
    def latent_dim(self):
        return self.channels * self.levels

    @classmethod
    def from_field(cls, field, device="cuda"):
        planes = [[_dev(p, device) for p in level] for level in field.planes]
        return cls(planes, field.aabb, field.channels)

    def zeros_like(self):
        return DeviceField([[torch.zeros_like(p) for p in level] for level in self.planes],
                           self.aabb, self.channels)

    def struct(self):
        h = N.HexPlane()
        h.levels = self.levels
        h.channels = self.channels
        if self.levels > N.MAX_LEVELS:
            raise ConfigurationError(f"at most {N.MAX_LEVELS} hexplane levels are supported")
        for l, level in enumerate(self.planes):
            for p, plane in enumerate(level):
                h.res[l][p][0] = plane.shape[0]
                h.res[l][p][1] = plane.shape[1]
                h.planes[l][p] = plane.data_ptr()
        h.aabb[:] = [float(v) for v in self.aabb.reshape(6)]
        h.order = _p(self.order)
        return h

    def with_order(self, order):
        """Same planes, visited in `order` (results are identical)."""
        return DeviceField(self.planes, self.aabb, self.channels, order)


class DeviceNet:
    """Deformation MLP weights ([out,in] fp32, exactly LinearLayer.weight)."""

    def __init__(self, layers, latent_dim, width, depth, feature_dim, enable_grid=True,
                 enable_feature_update=True):
        # layers: dict stack-name -> list of (weight, bias, relu)
        self.layers = layers
        self.latent_dim = int(latent_dim)
        self.width = int(width)
        self.depth = int(depth)
        self.feature_dim = int(feature_dim)
        self.enable_grid = bool(enable_grid)
        self.enable_feature_update = bool(enable_feature_update)

    @staticmethod
    def stack_names():
        names = ["net.trunk"]
        for b in BRANCHES:
            names += [f"net.ext.{b}", f"net.head.{b}"]
        return names + ["net.feat"]

    @classmethod
    def from_net(cls, net, device="cuda"):
        layers = {}
        for prefix, stack in net.stacks():
            layers[prefix] = [(_dev(l.weight, device), _dev(l.bias, device),
                               l.activation == "relu") for l in stack]
        c = net.cfg
        return cls(layers, net.latent_dim, c.width, c.depth, c.feature_dim, c.enable_grid,
                   c.enable_feature_update)

    def zeros_like(self):
        layers = {k: [(torch.zeros_like(w), torch.zeros_like(b), r) for (w, b, r) in v]
                  for k, v in self.layers.items()}
        return DeviceNet(layers, self.latent_dim, self.width, self.depth, self.feature_dim,
                         self.enable_grid, self.enable_feature_update)

    def struct(self):
        s = N.DeformNet()
        s.latent_dim = self.latent_dim
        s.width = self.width
        s.depth = self.depth
        s.feature_dim = self.feature_dim
        s.enable_grid = int(self.enable_grid)
        s.enable_feature_update = int(self.enable_feature_update)
        if self.depth > N.MAX_TRUNK:
            raise ConfigurationError(f"trunk depth above {N.MAX_TRUNK} is not supported")

        def fill(dst, layer):
            w, b, relu = layer
            dst.weight = w.data_ptr()
            dst.bias = b.data_ptr()
            dst.out_dim, dst.in_dim = int(w.shape[0]), int(w.shape[1])
            dst.relu = int(relu)

        for i, layer in enumerate(self.layers["net.trunk"]):
            fill(s.trunk[i], layer)
        for bi, b in enumerate(BRANCHES):
            for k in range(2):
                fill(s.ext[bi][k], self.layers[f"net.ext.{b}"][k])
            fill(s.head[bi], self.layers[f"net.head.{b}"][0])
        for k in range(2):
            fill(s.feat[k], self.layers["net.feat"][k])
        return s


def locality_order(positions, aabb, device="cuda"):
    """fs4d_locality_order: int32 [K] Morton order of `positions` ([K,3] fp32
    CUDA) inside `aabb` -- a model-load-time permutation for
    DeviceField.order (never changes results, only cache locality)."""
    lib = N.load()
    k = int(positions.shape[0])
    order = torch.empty(max(k, 1), dtype=torch.int32, device=device)
    ws = torch.empty(max(int(lib.fs4d_locality_order_workspace_bytes(k)), 1), dtype=torch.uint8, device=device)
    box = (ctypes.c_double * 6)(*[float(v) for v in np.asarray(aabb, dtype=np.float64).reshape(6)])
    N.check(lib.fs4d_locality_order(_p(positions), k, box, _p(order), _p(ws), ws.numel(), _stream()))
    return order[:k]


class DeformCache:
    """Device counterpart of deform_with_cache's `cache` (deformation.py:105):
    the tensor-core operand images of every MLP activation, written by
    DeformEngine.forward(with_cache=...) and read by DeformEngine.backward.
    Empty (0 bytes) when the net is outside the tensor-core backward, whose
    fallback recomputes the forward."""

    def __init__(self, nbytes, device):
        self.buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
        self.nbytes = int(nbytes)
        self.t = None
        self.k = None

    def ptr(self):
        return self.buf.data_ptr() if self.nbytes else None


class DeformEngine:
    """Runs fs4d_deform_fwd / fs4d_deform_bwd with a cached workspace."""

    def __init__(self, device="cuda"):
        self.device = device
        self.ws = None

    def cache_bytes(self, net, field, k):
        return int(N.load().fs4d_deform_cache_bytes(ctypes.byref(net.struct()), ctypes.byref(field.struct()), k))

    def _workspace(self, net_s, k):
        need = N.load().fs4d_deform_workspace_bytes(ctypes.byref(net_s), k)
        if need == 0:
            N.check(N.ERR_CONFIG)
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(int(need), dtype=torch.uint8, device=self.device)
        return self.ws

    def forward(self, cloud, field, net, t, out=None, with_cache=None):
        """Snapshot at time t (raw-space deltas; colours/SH aliased).
        with_cache=True (or a DeformCache to reuse) is deform_with_cache:
        returns (snapshot, cache)."""
        k = len(cloud)
        cache = None
        if with_cache is not None and with_cache is not False:
            need = self.cache_bytes(net, field, k)
            cache = with_cache if isinstance(with_cache, DeformCache) else None
            if cache is None or cache.buf.numel() < need:
                cache = DeformCache(need, self.device)
            cache.nbytes = need
            cache.t, cache.k = float(t), k
        if out is None:
            out = DeviceCloud.empty(k, cloud.feature_dim, 0, self.device)
        out.colors_raw = cloud.colors_raw
        out.sh_rest = cloud.sh_rest
        if not net.enable_feature_update:
            out.features = cloud.features
        cs, fs, ns, os_ = cloud.struct(), field.struct(), net.struct(), out.struct()
        ws = self._workspace(ns, k)
        cptr, cbytes = (cache.ptr(), cache.nbytes) if cache is not None else (None, 0)
        N.check(N.load().fs4d_deform_fwd(ctypes.byref(cs), ctypes.byref(fs), ctypes.byref(ns),
                                         float(t), ctypes.byref(os_), cptr, cbytes, _p(ws), ws.numel(),
                                         None, _stream()))
        return (out, cache) if cache is not None else out

    def backward(self, cloud, field, net, t, snap_grads, cloud_grads=None, net_grads=None,
                 plane_grads=None, accumulate=False, cache=None, deterministic=False, pass_event=None):
        """deform_backward on device.  Without output buffers: returns
        (d_positions [K,3], net_grads DeviceNet, plane_grads DeviceField|None).
        With a DeviceCloud `cloud_grads` (+ net/plane grads) every cloud
        gradient is written (or added, accumulate=True) and the buffers are
        returned.  deterministic=True: fs4d_deform_bwd_deterministic
        (fixed-point plane scatter, bitwise reproducible; needs `cache`).
        pass_event: a torch.cuda.Event recorded as soon as every cloud
        gradient except positions is written (fs4d_deform_bwd_split), for an
        all-reduce of those rows that overlaps the rest of the backward."""
        k = len(cloud)
        ngrads = net_grads if net_grads is not None else net.zeros_like()
        pgrads = plane_grads if plane_grads is not None else (field.zeros_like() if net.enable_grid else None)
        cs, fs, ns = cloud.struct(), field.struct(), net.struct()
        sgs, ngs = snap_grads.struct(), ngrads.struct()
        if cloud_grads is None:
            gpos = torch.empty(k, 3, dtype=torch.float32, device=self.device)
            cgs = N.Cloud()
            cgs.K = k
            cgs.positions = gpos.data_ptr()
        else:
            gpos = cloud_grads.positions
            cgs = cloud_grads.struct()
        pgs = pgrads.struct() if pgrads is not None else None
        ws = self._workspace(ns, k)
        if cache is not None and (cache.k != k or cache.t != float(t)):
            raise ContractViolation("deform cache was made for another (cloud, t)")
        cptr, cbytes = (cache.ptr(), cache.nbytes) if cache is not None else (None, 0)
        det_ws = None
        if deterministic:
            lib = N.load()
            need = int(lib.fs4d_deform_bwd_det_workspace_bytes(ctypes.byref(ns), ctypes.byref(fs)))
            if need == 0:
                raise ConfigurationError("the deterministic deform backward needs the tensor-core path (width 64, "
                                         "depth 1, levels * channels = 64, feature_dim <= 16)")
            if getattr(self, "det_ws", None) is None or self.det_ws.numel() < need:
                self.det_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            det_ws = self.det_ws
        if pass_event is not None:
            pass_event.record()  # materialise the cudaEvent_t (torch creates it lazily)
            N.check(N.load().fs4d_deform_bwd_split(
                ctypes.byref(cs), ctypes.byref(fs), ctypes.byref(ns), float(t), cptr, cbytes, ctypes.byref(sgs),
                ctypes.byref(cgs), ctypes.byref(ngs), ctypes.byref(pgs) if pgs is not None else None,
                int(bool(accumulate)), _p(ws), ws.numel(), _p(det_ws) if det_ws is not None else None,
                det_ws.numel() if det_ws is not None else 0, ctypes.c_void_p(pass_event.cuda_event), None,
                _stream()))
        elif deterministic:
            N.check(lib.fs4d_deform_bwd_deterministic(
                ctypes.byref(cs), ctypes.byref(fs), ctypes.byref(ns), float(t), cptr, cbytes, ctypes.byref(sgs),
                ctypes.byref(cgs), ctypes.byref(ngs), ctypes.byref(pgs) if pgs is not None else None,
                int(bool(accumulate)), _p(ws), ws.numel(), _p(self.det_ws), self.det_ws.numel(), None, _stream()))
        else:
            N.check(N.load().fs4d_deform_bwd(ctypes.byref(cs), ctypes.byref(fs), ctypes.byref(ns),
                                             float(t), cptr, cbytes, ctypes.byref(sgs), ctypes.byref(cgs),
                                             ctypes.byref(ngs),
                                             ctypes.byref(pgs) if pgs is not None else None,
                                             int(bool(accumulate)), _p(ws), ws.numel(), None, _stream()))
        return (cloud_grads if cloud_grads is not None else gpos), ngrads, pgrads


class RenderRecordDev:
    """Device render record: workspace + the sizes it was laid out for."""

    def __init__(self, info, ws, status):
        self.info = info
        self.ws = ws
        self.status = status

    @property
    def n_visible(self):
        return int(self.status.read()[N.ST_N_VISIBLE])

    @property
    def n_pairs(self):
        st = self.status.read()
        return (int(st[N.ST_PAIRS_HI]) << 32) | (int(st[N.ST_PAIRS_LO]) & 0xFFFFFFFF)


class Renderer:
    """Owns one reusable record; fs4d_render_fwd / fs4d_render_bwd."""

    def __init__(self, device="cuda", pair_capacity=None):
        self.device = device
        self.cap = pair_capacity
        self.ws = None
        self.status = StatusBlock(device)
        self.info = None

    def _info(self, k, h, w, d, sh, cap):
        i = N.RecordInfo()
        i.K, i.height, i.width, i.D, i.sh_degree, i.tile, i.pair_capacity = k, h, w, d, sh, 16, cap
        return i

    def _prepare(self, k, h, w, d, sh, tile):
        if tile != 16:
            raise ConfigurationError("only tile = 16 is implemented on device")
        if self.cap is None:
            self.cap = max(1024, 8 * k)
        info = self._info(k, h, w, d, sh, self.cap)
        need = N.load().fs4d_render_workspace_bytes(ctypes.byref(info))
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(int(need), dtype=torch.uint8, device=self.device)
        self.info = info
        return info

    def alloc_images(self, h, w, d):
        f = dict(dtype=torch.float32, device=self.device)
        return {"color": torch.empty(h, w, 3, **f), "depth": torch.empty(h, w, **f),
                "feature": torch.empty(h, w, d, **f), "alpha": torch.empty(h, w, **f),
                "n_contrib": torch.empty(h, w, dtype=torch.int32, device=self.device)}

    def forward(self, cloud, K, T, height, width, cfg, images=None, check=True):
        """Render one frame.  check=True reads the status block back (one
        sync) and raises / grows the pair buffer; check=False keeps the call
        fully asynchronous (caller checks self.status later)."""
        k, d, sh = len(cloud), cloud.feature_dim, cloud.sh_degree
        dout = d if cfg.with_features else 0
        if images is None:
            images = self.alloc_images(height, width, dout)
        cs, cam, rc = cloud.struct(), camera_struct(K, T, height, width), raster_struct(cfg)
        imgs = N.Images()
        imgs.color, imgs.depth, imgs.alpha = (images["color"].data_ptr(), images["depth"].data_ptr(),
                                              images["alpha"].data_ptr())
        imgs.feature = images["feature"].data_ptr() if dout > 0 else None
        imgs.n_contrib = images["n_contrib"].data_ptr() if images.get("n_contrib") is not None else None
        for _attempt in range(4):
            info = self._prepare(k, height, width, d, sh, cfg.tile)
            self.status.reset()
            N.check(N.load().fs4d_render_fwd(ctypes.byref(cs), ctypes.byref(cam), ctypes.byref(rc),
                                             ctypes.byref(info), _p(self.ws), self.ws.numel(),
                                             ctypes.byref(imgs), _p(self.status.t), _stream()))
            if not check:
                break
            st = self.status.read()
            if int(st[N.ST_CODE]) == N.ERR_CAPACITY:
                pairs = (int(st[N.ST_PAIRS_HI]) << 32) | (int(st[N.ST_PAIRS_LO]) & 0xFFFFFFFF)
                if pairs >= 2 ** 31:
                    raise ConfigurationError("more than 2^31 tile pairs in one frame")
                self.cap = int(pairs * 1.25) + 1024
                continue
            N.raise_device_status(st)
            break
        rec = RenderRecordDev(self.info, self.ws, self.status)
        return images, rec

    def backward(self, cloud, K, T, height, width, cfg, rec, d_color=None, d_depth=None,
                 d_feature=None, d_alpha=None, grads=None, viewspace=True, deterministic=False):
        """render_backward on device.  viewspace=True: depth-ordered
        (index, norm) pairs like SnapshotGrads; False: none (and no global
        depth sort); "dense": norms per Gaussian ([K], -1 for culled, no depth
        sort) for ViewspaceGradStats.add_dense; a tensor: dense norms into it."""
        k, d, sh = len(cloud), cloud.feature_dim, cloud.sh_degree
        if grads is None:
            grads = DeviceCloud.empty(k, d, sh, self.device)
        dense = isinstance(viewspace, torch.Tensor) or viewspace == "dense"
        vs_index = torch.empty(max(k, 1), dtype=torch.int32, device=self.device) \
            if (viewspace is True) else None
        if isinstance(viewspace, torch.Tensor):
            vs_norm = viewspace
        else:
            vs_norm = torch.empty(max(k, 1), dtype=torch.float32, device=self.device) if viewspace else None
        cs, cam, rc, gs = cloud.struct(), camera_struct(K, T, height, width), raster_struct(cfg), grads.struct()
        up = N.ImageGrads()
        up.d_color, up.d_depth = _p(d_color), _p(d_depth)
        up.d_feature, up.d_alpha = _p(d_feature), _p(d_alpha)
        if deterministic:  # fs4d_render_bwd_deterministic: ordered partials, no float atomics
            lib = N.load()
            need = max(int(lib.fs4d_render_bwd_det_workspace_bytes(ctypes.byref(rec.info))), 1)
            if getattr(self, "det_ws", None) is None or self.det_ws.numel() < need:
                self.det_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            N.check(lib.fs4d_render_bwd_deterministic(ctypes.byref(cs), ctypes.byref(cam), ctypes.byref(rc),
                                                      ctypes.byref(rec.info), _p(rec.ws), rec.ws.numel(),
                                                      ctypes.byref(up), ctypes.byref(gs), _p(vs_index), _p(vs_norm),
                                                      _p(self.det_ws), self.det_ws.numel(), None, _stream()))
        else:
            N.check(N.load().fs4d_render_bwd(ctypes.byref(cs), ctypes.byref(cam), ctypes.byref(rc),
                                             ctypes.byref(rec.info), _p(rec.ws), rec.ws.numel(),
                                             ctypes.byref(up), ctypes.byref(gs), _p(vs_index),
                                             _p(vs_norm), None, _stream()))
        if dense:
            return grads, None, vs_norm
        return grads, vs_index, vs_norm

    def export_projected(self, rec):
        k = int(rec.info.K)
        f = dict(dtype=torch.float32, device=self.device)
        out = {"mean2d": torch.zeros(k, 2, **f), "cov2d": torch.zeros(k, 3, **f),
               "conic": torch.zeros(k, 3, **f), "view_depth": torch.zeros(k, **f),
               "radius": torch.zeros(k, **f), "color": torch.zeros(k, 3, **f),
               "opacity": torch.zeros(k, **f),
               "source_index": torch.zeros(k, dtype=torch.int32, device=self.device),
               "tiles_touched": torch.zeros(k, dtype=torch.int32, device=self.device)}
        p = N.Projected()
        for name, t in out.items():
            setattr(p, name, t.data_ptr() if t.numel() else None)
        N.check(N.load().fs4d_render_export_projected(ctypes.byref(rec.info), _p(rec.ws),
                                                      rec.ws.numel(), ctypes.byref(p), _stream()))
        return out

    def export_tiles(self, rec):
        h, w = int(rec.info.height), int(rec.info.width)
        ntiles = ((h + 15) // 16) * ((w + 15) // 16)
        npairs = min(rec.n_pairs, int(rec.info.pair_capacity))
        ranges = torch.zeros(ntiles, 2, dtype=torch.int32, device=self.device)
        rows = torch.zeros(max(npairs, 1), dtype=torch.int32, device=self.device)
        N.check(N.load().fs4d_render_export_tiles(ctypes.byref(rec.info), _p(rec.ws), rec.ws.numel(),
                                                  _p(ranges), _p(rows), npairs, _stream()))
        return ranges, rows[:npairs]


STAGES = ("deform_fwd", "preprocess", "depth_sort", "binning", "blend", "blend_bwd",
          "preprocess_bwd", "deform_bwd", "deform_gather", "deform_mlp")


def profile_enable(on=True):
    N.load().fs4d_profile_enable(int(bool(on)))


def profile_collect():
    """{stage: (total_ms, calls)} for the stages recorded since the last collect."""
    n = len(STAGES)
    ms = (ctypes.c_double * n)()
    calls = (ctypes.c_int64 * n)()
    N.check(N.load().fs4d_profile_collect(ms, calls, n))
    return {STAGES[i]: (ms[i], int(calls[i])) for i in range(n)}


class FramePipeline:
    """One deformed + rendered frame per call, the cli.render_frame path
    (cli.py:58-61: model_snapshot -> render) with device-resident buffers.

    run(t, K, T)                       everything already in HBM
    run(t, K, T, host_in=..., host_out=...)  end-to-end: H2D of the canonical
        cloud from pinned host memory, deform + render, D2H of the images.
    """

    def __init__(self, cloud, field, net, height, width, cfg, device="cuda"):
        self.cloud, self.field, self.net = cloud, field, net
        self.h, self.w, self.cfg = int(height), int(width), cfg
        self.deformer = DeformEngine(device)
        self.renderer = Renderer(device)
        k, d = len(cloud), cloud.feature_dim
        self.snap = DeviceCloud.empty(k, d, 0, device)
        self.images = self.renderer.alloc_images(self.h, self.w, d if cfg.with_features else 0)

    def pinned_host_buffers(self):
        """Pinned host copies of the canonical cloud and the output images."""
        host_in = {n: getattr(self.cloud, n).cpu().pin_memory() for n in DeviceCloud.FIELDS}
        if self.cloud.sh_rest is not None:
            host_in["sh_rest"] = self.cloud.sh_rest.cpu().pin_memory()
        host_out = {n: torch.empty(t.shape, dtype=t.dtype).pin_memory() for n, t in self.images.items()}
        return host_in, host_out

    def h2d_bytes(self, host_in):
        return sum(t.numel() * t.element_size() for t in host_in.values())

    def d2h_bytes(self):
        return sum(t.numel() * t.element_size() for n, t in self.images.items() if n != "n_contrib")

    def _bind(self):
        """Build every ctypes argument once; steady-state frames then cost two
        ABI calls (+ a status reset) of host time."""
        lib = N.load()
        self.snap.colors_raw = self.cloud.colors_raw
        self.snap.sh_rest = self.cloud.sh_rest
        if not self.net.enable_feature_update:
            self.snap.features = self.cloud.features
        c = dict(cloud=self.cloud.struct(), field=self.field.struct(), net=self.net.struct(),
                 snap=self.snap.struct(), raster=raster_struct(self.cfg), imgs=N.Images())
        ws = self.deformer._workspace(c["net"], len(self.cloud))
        c["dws"], c["dws_n"] = ws.data_ptr(), ws.numel()
        im = self.images
        c["imgs"].color, c["imgs"].depth, c["imgs"].alpha = (im["color"].data_ptr(), im["depth"].data_ptr(),
                                                             im["alpha"].data_ptr())
        c["imgs"].feature = im["feature"].data_ptr() if im["feature"].numel() else None
        c["imgs"].n_contrib = im["n_contrib"].data_ptr()
        k, d, sh = len(self.snap), self.snap.feature_dim, self.snap.sh_degree
        c["info"] = self.renderer._prepare(k, self.h, self.w, d, sh, self.cfg.tile)
        c["rws"], c["rws_n"] = self.renderer.ws.data_ptr(), self.renderer.ws.numel()
        c["status"] = self.renderer.status.t.data_ptr()
        c["cap"] = self.renderer.cap
        c["cam_key"] = None
        self._c = c
        self._lib = lib

    def run(self, t, K, T, host_in=None, host_out=None, check=False):
        if host_in is not None:
            for n, src in host_in.items():
                getattr(self.cloud, n).copy_(src, non_blocking=True)
        c = getattr(self, "_c", None)
        if check or c is None or c["cap"] != self.renderer.cap:
            # checked path: sizes / grows the pair buffer, raises device errors
            self.deformer.forward(self.cloud, self.field, self.net, t, out=self.snap)
            self.renderer.forward(self.snap, K, T, self.h, self.w, self.cfg, images=self.images, check=check)
            self._bind()
        else:
            lib, s = self._lib, _stream()
            key = (np.asarray(K, dtype=np.float64).tobytes(), np.asarray(T, dtype=np.float64).tobytes())
            if key != c["cam_key"]:
                c["cam"] = camera_struct(K, T, self.h, self.w)
                c["cam_key"] = key
            N.check(lib.fs4d_deform_fwd(ctypes.byref(c["cloud"]), ctypes.byref(c["field"]), ctypes.byref(c["net"]),
                                        float(t), ctypes.byref(c["snap"]), None, 0, c["dws"], c["dws_n"], None, s))
            N.check(lib.fs4d_status_reset(c["status"], s))
            N.check(lib.fs4d_render_fwd(ctypes.byref(c["snap"]), ctypes.byref(c["cam"]), ctypes.byref(c["raster"]),
                                        ctypes.byref(c["info"]), c["rws"], c["rws_n"], ctypes.byref(c["imgs"]),
                                        c["status"], s))
        if host_out is not None:
            for n, dst in host_out.items():
                if n != "n_contrib":
                    dst.copy_(self.images[n], non_blocking=True)
        return self.images


class SequenceRenderer:
    """Render a timestep sequence (configs[2], cli.py:220-246) with several
    frames in flight: `pipelines` FramePipelines (own snapshot, render record,
    images), pipeline p always on stream p % streams, frames assigned round
    robin.  Consecutive frames are independent, so frame k+1's deformation
    runs on the SMs frame k's tile kernels leave idle.  `replicas` > 1 gives
    every pipeline its own copy of the model (the bench uses 4 so the model
    rotation exceeds L2 and no cache flush is needed between frames)."""

    def __init__(self, cloud, field, net, height, width, cfg, pipelines=2, streams=2, replicas=1, device="cuda"):
        # FS4D_SEQ_PRIO=1: stream i gets scheduling priority -i (clamped to the
        # device range), so one frame leads and the others fill its gaps
        prio = os.environ.get("FS4D_SEQ_PRIO", "0") == "1"
        lo, hi = torch.cuda.Stream.priority_range() if prio else (0, 0)
        self.streams = [torch.cuda.Stream(device=device, priority=max(hi, -i) if prio else 0) for i in range(streams)]
        self.pipes = []
        for p in range(pipelines):
            if replicas > 1 and p % replicas:
                c = DeviceCloud(*(getattr(cloud, n).clone() for n in DeviceCloud.FIELDS),
                                sh_rest=None if cloud.sh_rest is None else cloud.sh_rest.clone())
                f = DeviceField([[pl.clone() for pl in lv] for lv in field.planes], field.aabb, field.channels,
                                field.order)
                nt = DeviceNet({k: [(w.clone(), b.clone(), r) for (w, b, r) in v] for k, v in net.layers.items()},
                               net.latent_dim, net.width, net.depth, net.feature_dim, net.enable_grid,
                               net.enable_feature_update)
            else:
                c, f, nt = cloud, field, net
            self.pipes.append(FramePipeline(c, f, nt, height, width, cfg, device))

    def warm(self, t, K, T, pair_capacity=None):
        for p, pipe in enumerate(self.pipes):
            with torch.cuda.stream(self.streams[p % len(self.streams)]):
                pipe.run(t, K, T, check=True)
                if pair_capacity:
                    pipe.renderer.cap = max(pipe.renderer.cap, int(pair_capacity))
                pipe.run(t, K, T, check=True)
        torch.cuda.synchronize()

    def run(self, ts, K, T):
        """Enqueue one frame per t; returns (start, end) events on the current
        stream bracketing all of them."""
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(cur)
        for s in self.streams:
            s.wait_event(start)
        for i, t in enumerate(ts):
            p = i % len(self.pipes)
            with torch.cuda.stream(self.streams[p % len(self.streams)]):
                self.pipes[p].run(float(t), K, T)
        for s in self.streams:
            cur.wait_stream(s)
        end.record(cur)
        return start, end

    def raise_if_error(self):
        for pipe in self.pipes:
            pipe.renderer.status.raise_if_error()


class StreamedFrames:
    """End-to-end frame stream from host buffers with copy/compute overlap.

    Two FramePipeline replicas (own device cloud copy, render record and
    images) alternate over two CUDA streams, so frame i+1's host->device copy
    of the canonical cloud and frame i-1's device->host copy of the images run
    on the copy engines while frame i computes.  Every frame still performs
    its full H2D and D2H.
    """

    def __init__(self, cloud, field, net, height, width, cfg, device="cuda"):
        self.pipes = []
        self.streams = [torch.cuda.Stream(device=device) for _ in range(2)]
        for p in range(2):
            c = cloud if p == 0 else DeviceCloud(*(getattr(cloud, n).clone() for n in DeviceCloud.FIELDS),
                                                 sh_rest=None if cloud.sh_rest is None else cloud.sh_rest.clone())
            self.pipes.append(FramePipeline(c, field, net, height, width, cfg, device))
        self.host_in, out0 = self.pipes[0].pinned_host_buffers()
        _, out1 = self.pipes[1].pinned_host_buffers()
        self.host_out = [out0, out1]

    def warm(self, t, K, T):
        for p, pipe in enumerate(self.pipes):
            with torch.cuda.stream(self.streams[p]):
                pipe.run(t, K, T, check=True)
                pipe.run(t, K, T, host_in=self.host_in, host_out=self.host_out[p])
        torch.cuda.synchronize()

    def run(self, ts, K, T):
        """Enqueue one frame per t; returns (start_event, end_event) on the
        current stream bracketing the whole stream of frames."""
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(cur)
        for s in self.streams:
            s.wait_event(start)
        for i, t in enumerate(ts):
            p = i % 2
            with torch.cuda.stream(self.streams[p]):
                self.pipes[p].run(float(t), K, T, host_in=self.host_in, host_out=self.host_out[p])
        for s in self.streams:
            cur.wait_stream(s)
        end.record(cur)
        return start, end

    def h2d_bytes(self):
        return self.pipes[0].h2d_bytes(self.host_in)

    def d2h_bytes(self):
        return self.pipes[0].d2h_bytes()


# ---------------------------------------------------------------------------
# numpy <-> device helpers for the reference-shaped wrappers
# ---------------------------------------------------------------------------
def as_device(x, device="cuda"):
    """(fp32 contiguous CUDA tensor, came_from_host).  torch CUDA fp32 tensors
    pass through without a copy (the zero-copy fast path); anything else is a
    host array (the reference's float64 NumPy) rounded to fp32 and uploaded."""
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32:
        return x.contiguous(), False
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=torch.float32).contiguous(), True
    return _dev(x, device), True


def to_host(t, like_host):
    """Back to float64 NumPy when the caller passed host arrays (reference API);
    otherwise the device tensor itself."""
    return t.detach().cpu().numpy().astype(np.float64) if like_host else t
