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
        return self._proj

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
        """Contributing (source_index, alpha, weight) triples of one pixel,
        replayed from the record's projected Gaussians (rasterizer.py:102-114)."""
        rec = self.record
        t = rec.cfg.tile
        rows = rec.tile_lists()[row // t][col // t]
        if rows.size == 0:
            return np.empty(0, dtype=np.int64), np.empty(0), np.empty(0)
        proj = rec.proj
        cfg = rec.cfg
        src, alphas, weights = [], [], []
        T = 1.0
        q_skip = 2.0 * np.log(255.0)
        for g in rows:
            dx = col - proj.mean2d[g, 0]
            dy = row - proj.mean2d[g, 1]
            r = proj.radius[g]
            if abs(dx) > r or abs(dy) > r:
                continue
            c = proj.conic[g]
            q = c[0, 0] * dx * dx + (c[0, 1] + c[1, 0]) * dx * dy + c[1, 1] * dy * dy
            if q > q_skip:
                continue
            a = min(proj.opacity[g] * np.exp(-0.5 * q), cfg.alpha_cap)
            if a < cfg.alpha_skip:
                continue
            if T < cfg.stop_transmittance:
                break
            src.append(proj.source_index[g])
            alphas.append(a)
            weights.append(a * T)
            T *= 1.0 - a
        return (np.asarray(src, dtype=np.int64), np.asarray(alphas, dtype=np.float64),
                np.asarray(weights, dtype=np.float64))


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
                    dL_dalpha=None):
    """Gradients for every raw snapshot parameter (rasterizer.py:320-452)."""
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
        d_feature=up(dL_dfeature, (h, w, n)) if n else None, d_alpha=up(dL_dalpha, (h, w)))
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
