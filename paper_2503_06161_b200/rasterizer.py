"""Tile rasterizer on the GPU: the drop-in for featsplat.rasterizer
(rasterizer.py:26-452).

Same dataclasses and signatures, NumPy float64 in/out.  ``render`` is one
fs4d_render_fwd call (fp64 projection, stable depth radix sort, tile binning,
register-accumulated RGB + depth + D-feature blend); ``render_backward`` is
one fs4d_render_bwd call replaying the device record.  ``project`` and
``bin_tiles`` read the same record back.

Conventions are the reference's (rasterizer.py:12-15): pixel (row i, col j)
is sampled at (u=j, v=i); the square footprint of half-width ``radius`` gates
both binning and compositing; the Gaussian that drops T below the stop
threshold is composited.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError, ContractViolation


@dataclass
class RasterConfig:
    tile: int = 16
    z_near: float = 0.01
    lowpass: float = 0.3
    alpha_cap: float = 0.99
    alpha_skip: float = 1.0 / 255.0
    stop_transmittance: float = 1e-4
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    with_features: bool = True


@dataclass
class ProjectedGaussians:
    """Screen-space Gaussians, depth-sorted front to back (rasterizer.py:38-61)."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    view_depth: np.ndarray
    radius: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    feature: np.ndarray
    source_index: np.ndarray

    def __len__(self):
        return int(self.mean2d.shape[0])

    def __getitem__(self, i):
        return {"mean2d": self.mean2d[i], "cov2d": self.cov2d[i], "view_depth": self.view_depth[i],
                "radius": self.radius[i], "color": self.color[i], "opacity": self.opacity[i],
                "feature": self.feature[i], "source_index": self.source_index[i]}


@dataclass
class TileRecord:
    """Compositing state of one tile (rasterizer.py:64-78), replayed from the
    device record: depth-ordered rows into ``proj`` with at least one live
    pixel, and their [G, P] gated alpha, 2-d Gaussian and raw alpha values
    exactly as the blend kernel evaluated them."""

    rows: np.ndarray
    alpha: np.ndarray
    g2d: np.ndarray
    a_raw: np.ndarray
    x0: int
    y0: int
    xs: np.ndarray
    ys: np.ndarray


@dataclass
class RasterRecord:
    """Device record replayed by the backward (rasterizer.py:81-91)."""

    device: object       # device.RenderRecordDev
    renderer: object     # device.Renderer that owns the workspace
    height: int
    width: int
    cfg: RasterConfig
    snapshot_len: int
    feature_dim: int
    _proj: object = None
    _tiles: object = None

    @property
    def proj(self):
        if self._proj is None:
            self._proj = _export_projected(self)
            self._proj._record = self
        return self._proj

    @property
    def tiles(self):
        """Flat list of TileRecord for every tile with a live row, in the
        reference's row-major tile order (rasterizer.py:275-288), replayed on
        the device from this record (fs4d_render_tile_alphas)."""
        if getattr(self, "_tile_records", None) is None:
            t = self.cfg.tile
            recs = []
            for ty, row in enumerate(self.tile_lists()):
                ys = np.arange(ty * t, min(ty * t + t, self.height))
                for tx, idx in enumerate(row):
                    if idx.size == 0:
                        continue
                    xs = np.arange(tx * t, min(tx * t + t, self.width))
                    rows, alpha, g2d, a_raw = _tile_alphas(self.proj, idx, xs, ys, self.cfg)
                    if rows.size:
                        recs.append(TileRecord(rows=rows, alpha=alpha, g2d=g2d, a_raw=a_raw, x0=int(xs[0]),
                                               y0=int(ys[0]), xs=xs, ys=ys))
            self._tile_records = recs
        return self._tile_records

    def tile_lists(self):
        """tiles[ty][tx] -> rows into ``proj`` in depth order (bin_tiles layout)."""
        if self._tiles is None:
            ranges, rows = self.renderer.export_tiles(self.device)
            ranges = ranges.cpu().numpy().astype(np.int64)
            rows = rows.cpu().numpy().astype(np.int64)
            t = self.cfg.tile
            ntx, nty = -(-self.width // t), -(-self.height // t)
            self._tiles = [[rows[ranges[ty * ntx + tx, 0]:ranges[ty * ntx + tx, 1]]
                            for tx in range(ntx)] for ty in range(nty)]
        return self._tiles


@dataclass
class RenderOutput:
    color: np.ndarray
    depth: np.ndarray
    feature: np.ndarray
    alpha: np.ndarray
    record: RasterRecord
    n_contrib: np.ndarray = None   # live contributors per pixel (a19)

    def pixel_record(self, row, col):
        """Contributing (source_index, alpha, weight) triples of one pixel
        (rasterizer.py:102-114), replayed on the device from the render
        record with the blend kernel's arithmetic (fs4d_render_tile_alphas +
        fs4d_composite_weights), so they agree with ``n_contrib``."""
        rec = self.record
        t = rec.cfg.tile
        idx = rec.tile_lists()[row // t][col // t]
        empty = (np.empty(0, dtype=np.int64), np.empty(0), np.empty(0))
        if idx.size == 0:
            return empty
        y0, x0 = (row // t) * t, (col // t) * t
        xs = np.arange(x0, min(x0 + t, rec.width))
        ys = np.arange(y0, min(y0 + t, rec.height))
        rows, alpha, _, _ = _tile_alphas(rec.proj, idx, xs, ys, rec.cfg)
        if rows.size == 0:
            return empty
        p = (row - y0) * xs.size + (col - x0)
        _, contrib, w, _ = _composite_weights(alpha, rec.cfg.stop_transmittance)
        a = alpha[:, p]
        live = (a > 0) & contrib[:, p]
        return rec.proj.source_index[rows[live]], a[live], w[live, p]


@dataclass
class SnapshotGrads:
    positions: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    colors_raw: np.ndarray
    features: np.ndarray
    viewspace_index: np.ndarray
    viewspace_norm: np.ndarray
    sh_rest: np.ndarray = None


def _renderer():
    from .device import Renderer
    return Renderer()


def _host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _check_cfg(cfg):
    if cfg.tile != 16:
        raise ConfigurationError("only tile = 16 is implemented on device")


def _render_device(snapshot, frame, cfg):
    from .device import DeviceCloud
    _check_cfg(cfg)
    rnd = _renderer()
    dc = DeviceCloud.from_cloud(snapshot)
    images, rec = rnd.forward(dc, frame.K, frame.T, frame.height, frame.width, cfg, check=True)
    record = RasterRecord(device=rec, renderer=rnd, height=frame.height, width=frame.width,
                          cfg=cfg, snapshot_len=len(snapshot), feature_dim=snapshot.features.shape[1])
    record._snapshot_features = snapshot.features
    return images, record


def _export_projected(record):
    p = record.renderer.export_projected(record.device)
    m = record.device.n_visible
    src = p["source_index"][:m].cpu().numpy().astype(np.int64)
    cov = _host(p["cov2d"][:m])
    con = _host(p["conic"][:m])
    feats = record._snapshot_features
    n = feats.shape[1] if record.cfg.with_features else 0
    return ProjectedGaussians(
        mean2d=_host(p["mean2d"][:m]),
        cov2d=np.stack([cov[:, [0, 1]], cov[:, [1, 2]]], axis=1),
        conic=np.stack([con[:, [0, 1]], con[:, [1, 2]]], axis=1),
        view_depth=_host(p["view_depth"][:m]),
        radius=_host(p["radius"][:m]),
        color=_host(p["color"][:m]),
        opacity=_host(p["opacity"][:m]),
        feature=np.asarray(feats, dtype=np.float64)[src, :n] if n else np.zeros((m, 0)),
        source_index=src,
    )


def _tile_alphas(proj, idx, xs, ys, cfg):
    """Gated alpha matrices of one tile, compressed to rows that touch it
    (rasterizer.py:215-234): (rows, alpha, g2d, a_raw) with rows indexing into
    ``proj``.  Replayed on the device from the render record ``proj`` came
    from, with the blend kernel's own arithmetic; ``proj`` must come from
    this package's project() / render()."""
    import torch
    import ctypes

    from . import _native as N
    from .device import _p, _stream, raster_struct
    rec = getattr(proj, "_record", None)
    if rec is None:
        raise ContractViolation("_tile_alphas needs the ProjectedGaussians of a device project() / render() call")
    idx = np.asarray(idx, dtype=np.int64).reshape(-1)
    xs, ys = np.asarray(xs, dtype=np.int64), np.asarray(ys, dtype=np.int64)
    nx, ny = int(xs.size), int(ys.size)
    if (nx and not np.array_equal(xs, np.arange(xs[0], xs[0] + nx))) or \
            (ny and not np.array_equal(ys, np.arange(ys[0], ys[0] + ny))):
        raise ConfigurationError("tile pixel columns / rows must be contiguous ranges")
    g = int(idx.size)
    if g == 0 or nx == 0 or ny == 0:
        z = np.zeros((0, nx * ny))
        return idx[:0], z, z.copy(), z.copy()
    dev = rec.device
    src = torch.as_tensor(proj.source_index[idx].astype(np.int32), device="cuda")
    f = dict(dtype=torch.float32, device="cuda")
    alpha, g2d, a_raw = torch.empty(g, nx * ny, **f), torch.empty(g, nx * ny, **f), torch.empty(g, nx * ny, **f)
    rc = raster_struct(rec.cfg if cfg is None else cfg)
    N.check(N.load().fs4d_render_tile_alphas(ctypes.byref(dev.info), _p(dev.ws), dev.ws.numel(), ctypes.byref(rc),
                                             _p(src), g, int(xs[0]), int(ys[0]), nx, ny, _p(alpha), _p(g2d),
                                             _p(a_raw), _stream()))
    alpha, g2d, a_raw = _host(alpha), _host(g2d), _host(a_raw)
    keep = np.nonzero(alpha.max(axis=1) > 0.0)[0]
    return idx[keep], alpha[keep], g2d[keep], a_raw[keep]


def _composite_weights(alpha, stop):
    """(t_exc, contrib, w, t_final) of a [G, P] alpha matrix
    (rasterizer.py:244-261), front to back on the device in fp32 with the
    blend kernel's multiplication order."""
    import torch

    from . import _native as N
    from .device import _p, _stream, as_device
    a, _ = as_device(np.atleast_2d(np.asarray(alpha, dtype=np.float64)) if not isinstance(alpha, torch.Tensor)
                     else alpha)
    g, p = int(a.shape[0]), int(a.shape[1])
    f = dict(dtype=torch.float32, device=a.device)
    t_exc, w = torch.empty(g, p, **f), torch.empty(g, p, **f)
    contrib = torch.empty(g, p, dtype=torch.uint8, device=a.device)
    t_final = torch.empty(p, **f)
    N.check(N.load().fs4d_composite_weights(_p(a), g, p, float(stop), _p(t_exc), _p(contrib), _p(w), _p(t_final),
                                            _stream()))
    return _host(t_exc), contrib.cpu().numpy().astype(bool), _host(w), _host(t_final)


def project(snapshot, frame, cfg):
    """Projected, culled, depth-sorted Gaussians (rasterizer.py:117-185)."""
    _, record = _render_device(snapshot, frame, cfg)
    proj = record.proj
    proj._record = record
    return proj


def bin_tiles(proj, height, width, tile):
    """Per-tile depth-ordered rows into ``proj`` (rasterizer.py:188-207).
    ``proj`` must come from :func:`project` (the lists are the device's)."""
    rec = getattr(proj, "_record", None)
    if rec is None or rec.height != height or rec.width != width or rec.cfg.tile != tile:
        raise ContractViolation("bin_tiles needs the ProjectedGaussians of a device project() "
                                "call with the same image size and tile")
    return rec.tile_lists()


def render(snapshot, frame, cfg):
    """Composite colour, depth, features and alpha for one frame (rasterizer.py:264-303)."""
    images, record = _render_device(snapshot, frame, cfg)
    h, w = frame.height, frame.width
    n = snapshot.features.shape[1] if cfg.with_features else 0
    return RenderOutput(
        color=_host(images["color"]).reshape(h, w, 3),
        depth=_host(images["depth"]).reshape(h, w),
        feature=_host(images["feature"]).reshape(h, w, n) if n else np.zeros((h, w, 0)),
        alpha=_host(images["alpha"]).reshape(h, w),
        record=record,
        n_contrib=images["n_contrib"].cpu().numpy().astype(np.int64),
    )


def render_backward(snapshot, frame, out, dL_dcolor=None, dL_ddepth=None, dL_dfeature=None,
                    dL_dalpha=None, *, deterministic=False):
    """Gradients for every raw snapshot parameter (rasterizer.py:320-452).
    deterministic=True (extension): fixed-order reduction instead of float
    atomics, bitwise reproducible (fs4d_render_bwd_deterministic)."""
    import torch
    from .device import DeviceCloud

    rec = out.record
    h, w = rec.height, rec.width
    if rec.snapshot_len != len(snapshot) or (frame.height, frame.width) != (h, w):
        raise ContractViolation("record does not match this snapshot/frame")
    n = snapshot.features.shape[1] if rec.cfg.with_features else 0
    if dL_dfeature is not None and np.shape(dL_dfeature) != (h, w, n):
        raise ContractViolation(f"dL_dfeature must have shape {(h, w, n)}")

    def up(x, shape):
        if x is None:
            return None
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device="cuda").reshape(shape)

    dc = DeviceCloud.from_cloud(snapshot)
    grads, vs_index, vs_norm = rec.renderer.backward(
        dc, frame.K, frame.T, h, w, rec.cfg, rec.device,
        d_color=up(dL_dcolor, (h, w, 3)), d_depth=up(dL_ddepth, (h, w)),
        d_feature=up(dL_dfeature, (h, w, n)) if n else None, d_alpha=up(dL_dalpha, (h, w)),
        deterministic=deterministic)
    k = len(snapshot)
    m = rec.device.n_visible
    sh = getattr(snapshot, "sh_rest", None)
    return SnapshotGrads(
        positions=_host(grads.positions).reshape(k, 3),
        rotations=_host(grads.rotations).reshape(k, 4),
        log_scales=_host(grads.log_scales).reshape(k, 3),
        opacity_logits=_host(grads.opacity_logits).reshape(k),
        colors_raw=_host(grads.colors_raw).reshape(k, 3),
        features=_host(grads.features).reshape(k, np.shape(snapshot.features)[1]),
        viewspace_index=vs_index[:m].cpu().numpy().astype(np.int64),
        viewspace_norm=_host(vs_norm[:m]),
        sh_rest=None if sh is None else _host(grads.sh_rest).reshape(np.shape(sh)),
    )
