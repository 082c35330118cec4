"""CPU float64 oracle for the FE-4DGS render path — TEST INFRASTRUCTURE ONLY.

This module is the checker the GPU path is compared against.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu-baseline / reference arm may import
it; the product package (paper_2503_06161_b200) never does, and has no CPU
fallback.

It is a NumPy float64 restatement of the reference algorithm
(/root/reference/pkg/src/featsplat, package `featsplat` 0.1.0), written
independently; every function cites the reference lines it follows.  It is
pinned against golden vectors produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle_golden.py).  The SH > 0 colour term is the build's own
extension and is *parity-unpinned* (the reference is degree-0 only,
SPEC.md:172); at degree 0 it reduces exactly to the reference.

Inputs are duck-typed: any object with the GaussianCloud attribute names
(positions, rotations, log_scales, opacity_logits, colors_raw, features and
optionally sh_rest) works.
"""

import numpy as np

Q_SKIP = 2.0 * np.log(255.0)  # rasterizer.py:212
PLANE_AXES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))  # hexplane.py:16
BRANCHES = ("position", "rotation", "scale", "opacity")  # deformation.py:19
BRANCH_DIMS = (3, 4, 3, 1)  # deformation.py:20


class OracleError(Exception):
    """Raised where the reference raises (kind in .kind: numeric/data/degenerate/contract)."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


class RasterParams:
    """RasterConfig defaults (rasterizer.py:26-35)."""

    def __init__(self, tile=16, z_near=0.01, lowpass=0.3, alpha_cap=0.99, alpha_skip=1.0 / 255.0,
                 stop_transmittance=1e-4, background=(0.0, 0.0, 0.0), with_features=True):
        self.tile = tile
        self.z_near = z_near
        self.lowpass = lowpass
        self.alpha_cap = alpha_cap
        self.alpha_skip = alpha_skip
        self.stop_transmittance = stop_transmittance
        self.background = np.asarray(background, dtype=np.float64)
        self.with_features = with_features


# ---------------------------------------------------------------------------
# Gaussian math (gaussians.py:25-31, 140-218)
# ---------------------------------------------------------------------------
def sigmoid(x):
    """gaussians.py:25-31 — evaluated on |x| to avoid overflow."""
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(-np.abs(x))
    return np.where(x >= 0.0, 1.0 / (1.0 + e), e / (1.0 + e))


def unit_quats(q):
    """gaussians.py:174-178."""
    n = np.sqrt((q * q).sum(axis=1))
    if np.any(n < 1e-12):
        raise OracleError("degenerate", "quaternion norm below 1e-12")
    return q / n[:, None], n


def rotation_from_unit_quats(u):
    """gaussians.py:140-153 (w, x, y, z)."""
    w, x, y, z = (u[:, i] for i in range(4))
    R = np.empty((u.shape[0], 3, 3))
    R[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
    R[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
    R[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
    return R


def covariances(quats, log_scales):
    """Sigma = (R S)(R S)^T, gaussians.py:187-194."""
    u, _ = unit_quats(quats)
    R = rotation_from_unit_quats(u)
    A = R * np.exp(log_scales)[:, None, :]
    return np.einsum("kij,klj->kil", A, A)


def covariance_grads(quats, log_scales, dsigma):
    """gaussians.py:156-171, 181-184, 203-218."""
    u, n = unit_quats(quats)
    R = rotation_from_unit_quats(u)
    d = np.exp(2.0 * log_scales)
    sym = dsigma + np.transpose(dsigma, (0, 2, 1))
    dR = np.einsum("kij,kjl->kil", sym, R * d[:, None, :])
    diag = np.einsum("kji,kjl,kli->ki", R, dsigma, R)
    dls = 2.0 * d * diag
    w, x, y, z = (u[:, i] for i in range(4))
    g = dR.reshape(-1, 9)
    dw = 2 * (-z * g[:, 1] + y * g[:, 2] + z * g[:, 3] - x * g[:, 5] - y * g[:, 6] + x * g[:, 7])
    dx = 2 * (y * g[:, 1] + z * g[:, 2] + y * g[:, 3] - 2 * x * g[:, 4] - w * g[:, 5]
              + z * g[:, 6] + w * g[:, 7] - 2 * x * g[:, 8])
    dy = 2 * (-2 * y * g[:, 0] + x * g[:, 1] + w * g[:, 2] + x * g[:, 3] + z * g[:, 5]
              - w * g[:, 6] + z * g[:, 7] - 2 * y * g[:, 8])
    dz = 2 * (-2 * z * g[:, 0] - w * g[:, 1] + x * g[:, 2] + w * g[:, 3] - 2 * z * g[:, 4]
              + y * g[:, 5] + x * g[:, 6] + y * g[:, 7])
    du = np.stack([dw, dx, dy, dz], axis=1)
    dq = (du - (du * u).sum(axis=1, keepdims=True) * u) / n[:, None]
    return dq, dls


# ---------------------------------------------------------------------------
# SH extension (build-defined, parity-unpinned; degree 0 == reference)
# ---------------------------------------------------------------------------
_C1 = 0.4886025119029199
_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
       0.5462742152960396)
_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
       -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def sh_basis(degree, d):
    """Real SH bands 1..degree at unit directions d [N,3] -> [N, (L+1)^2-1]."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    cols = []
    if degree >= 1:
        cols += [-_C1 * y, _C1 * z, -_C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [_C2[0] * x * y, _C2[1] * y * z, _C2[2] * (2 * zz - xx - yy), _C2[3] * x * z,
                 _C2[4] * (xx - yy)]
    if degree >= 3:
        cols += [_C3[0] * y * (3 * xx - yy), _C3[1] * x * y * z, _C3[2] * y * (4 * zz - xx - yy),
                 _C3[3] * z * (2 * zz - 3 * xx - 3 * yy), _C3[4] * x * (4 * zz - xx - yy),
                 _C3[5] * z * (xx - yy), _C3[6] * x * (xx - 3 * yy)]
    if not cols:
        return np.zeros((d.shape[0], 0))
    return np.stack(cols, axis=1)


def sh_degree_of(cloud):
    sh = getattr(cloud, "sh_rest", None)
    if sh is None or np.shape(sh)[1] == 0:
        return 0
    return int(round(np.sqrt(np.shape(sh)[1] + 1))) - 1


def view_dirs(positions, T):
    """Unit vectors from the camera centre C = -R^T t to each position."""
    R, t = T[:3, :3], T[:3, 3]
    v = positions - (-(R.T @ t))[None, :]
    n = np.sqrt((v * v).sum(axis=1))
    n = np.where(n > 0, n, 1.0)
    return v / n[:, None], n


def raw_colors(cloud, idx, T):
    """Pre-clip colour: colors_raw (+ SH bands).  Reference: rasterizer.py:181."""
    base = np.asarray(cloud.colors_raw, dtype=np.float64)[idx]
    deg = sh_degree_of(cloud)
    if deg == 0:
        return base
    d, _ = view_dirs(np.asarray(cloud.positions, dtype=np.float64)[idx], T)
    Y = sh_basis(deg, d)
    sh = np.asarray(cloud.sh_rest, dtype=np.float64)[idx]
    return base + np.einsum("nk,nkc->nc", Y, sh)


# ---------------------------------------------------------------------------
# projection (rasterizer.py:117-185)
# ---------------------------------------------------------------------------
def project(cloud, K, T, height, width, cfg):
    """Returns a dict of depth-sorted projected Gaussians plus the fp64
    deciding quantities used by the margin-aware parity checks."""
    for name in ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw",
                 "features"):
        a = np.asarray(getattr(cloud, name), dtype=np.float64)
        bad = ~np.isfinite(a.reshape(a.shape[0], -1)).all(axis=1)
        if bad.any():
            raise OracleError("numeric", f"non-finite {name} for Gaussian indices "
                                         f"{np.flatnonzero(bad)[:8].tolist()}")
    K = np.asarray(K, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    if abs(K[0, 1]) > 1e-9:
        raise OracleError("data", "intrinsics with skew are not supported")
    pos = np.asarray(cloud.positions, dtype=np.float64)
    R, tv = T[:3, :3], T[:3, 3]
    cam = pos @ R.T + tv
    front = np.flatnonzero(cam[:, 2] > cfg.z_near)
    x, y, z = cam[front, 0], cam[front, 1], cam[front, 2]
    fx, fy, cx, cy = K[0, 0], K[1, 1], K[0, 2], K[1, 2]
    u = fx * x / z + cx
    v = fy * y / z + cy
    sig = covariances(np.asarray(cloud.rotations, dtype=np.float64)[front],
                      np.asarray(cloud.log_scales, dtype=np.float64)[front])
    J = np.zeros((front.size, 2, 3))
    J[:, 0, 0], J[:, 0, 2] = fx / z, -fx * x / (z * z)
    J[:, 1, 1], J[:, 1, 2] = fy / z, -fy * y / (z * z)
    M = J @ R
    c2 = M @ sig @ np.transpose(M, (0, 2, 1))
    c2[:, 0, 0] += cfg.lowpass
    c2[:, 1, 1] += cfg.lowpass
    a, b, c = c2[:, 0, 0], c2[:, 0, 1], c2[:, 1, 1]
    half_tr = 0.5 * (a + c)
    det = a * c - b * b
    lam = half_tr + np.sqrt(np.maximum(half_tr * half_tr - det, 0.0))
    rad_arg = 3.0 * np.sqrt(lam)
    radius = np.ceil(rad_arg)
    visible = (u + radius >= 0) & (u - radius <= width - 1) & (v + radius >= 0) & (v - radius <= height - 1)
    kept = np.flatnonzero(visible)
    order = kept[np.argsort(z[kept], kind="stable")]
    src = front[order]
    ck = c2[order]
    dk = det[order]
    conic = np.empty_like(ck)
    conic[:, 0, 0] = ck[:, 1, 1] / dk
    conic[:, 0, 1] = -ck[:, 0, 1] / dk
    conic[:, 1, 0] = -ck[:, 1, 0] / dk
    conic[:, 1, 1] = ck[:, 0, 0] / dk
    feats = np.asarray(cloud.features, dtype=np.float64)
    n = feats.shape[1] if cfg.with_features else 0
    raw = raw_colors(cloud, src, T)
    return {
        "mean2d": np.stack([u[order], v[order]], axis=1),
        "cov2d": ck,
        "conic": conic,
        "view_depth": z[order],
        "radius": radius[order],
        "color": np.clip(raw, 0.0, 1.0),
        "color_raw": raw,
        "opacity": sigmoid(np.asarray(cloud.opacity_logits, dtype=np.float64)[src]),
        "feature": feats[src, :n] if n else np.zeros((src.size, 0)),
        "source_index": src,
        # deciding quantities for margins (all front Gaussians, by source index)
        "front_index": front,
        "front_radius_arg": rad_arg,
        "front_z": z,
        "front_u": u,
        "front_v": v,
    }


def tile_rects(proj, height, width, tile):
    """Inclusive tile rectangle per projected Gaussian (rasterizer.py:192-201)."""
    ntx, nty = -(-width // tile), -(-height // tile)
    u, v, r = proj["mean2d"][:, 0], proj["mean2d"][:, 1], proj["radius"]
    tx0 = np.clip(np.floor((u - r) / tile).astype(np.int64), 0, ntx - 1)
    tx1 = np.clip(np.floor((u + r) / tile).astype(np.int64), 0, ntx - 1)
    ty0 = np.clip(np.floor((v - r) / tile).astype(np.int64), 0, nty - 1)
    ty1 = np.clip(np.floor((v + r) / tile).astype(np.int64), 0, nty - 1)
    return tx0, tx1, ty0, ty1


def bin_tiles(proj, height, width, tile):
    """tiles[ty][tx] -> depth-ordered rows (rasterizer.py:188-207), built by
    a stable sort of (tile id) over rows emitted in depth order."""
    ntx, nty = -(-width // tile), -(-height // tile)
    tx0, tx1, ty0, ty1 = tile_rects(proj, height, width, tile)
    span_x = tx1 - tx0 + 1
    counts = span_x * (ty1 - ty0 + 1)
    rows = np.repeat(np.arange(tx0.size, dtype=np.int64), counts)
    local = np.arange(rows.size, dtype=np.int64) - np.repeat(np.cumsum(counts) - counts, counts)
    ids = (ty0[rows] + local // span_x[rows]) * ntx + tx0[rows] + local % span_x[rows]
    perm = np.argsort(ids, kind="stable")
    ids, rows = ids[perm], rows[perm]
    bounds = np.searchsorted(ids, np.arange(ntx * nty + 1))
    return [[rows[bounds[ty * ntx + tx]:bounds[ty * ntx + tx + 1]] for tx in range(ntx)]
            for ty in range(nty)]


# ---------------------------------------------------------------------------
# compositing (rasterizer.py:210-303)
# ---------------------------------------------------------------------------
def tile_alpha(proj, rows, xs, ys, cfg):
    """Gated alphas [G, P] of one tile (rasterizer.py:215-241)."""
    px = np.tile(xs, ys.size).astype(np.float64)
    py = np.repeat(ys, xs.size).astype(np.float64)
    dx = px[None, :] - proj["mean2d"][rows, 0:1]
    dy = py[None, :] - proj["mean2d"][rows, 1:2]
    r = proj["radius"][rows][:, None]
    con = proj["conic"][rows]
    q = (con[:, 0, 0, None] * dx * dx + (con[:, 0, 1, None] + con[:, 1, 0, None]) * dx * dy
         + con[:, 1, 1, None] * dy * dy)
    inside = (np.abs(dx) <= r) & (np.abs(dy) <= r) & (q <= Q_SKIP)
    g = np.where(inside, np.exp(-0.5 * np.where(inside, q, 0.0)), 0.0)
    a_raw = proj["opacity"][rows][:, None] * g
    alpha = np.minimum(a_raw, cfg.alpha_cap)
    alpha = np.where(alpha < cfg.alpha_skip, 0.0, alpha)
    return alpha, g, a_raw, dx, dy, q, inside


def transmittance(alpha, stop):
    """Front-to-back bookkeeping (rasterizer.py:244-261): T before each row,
    contribution mask (T_before >= stop), weights, and T after the halt."""
    t_after = np.cumprod(1.0 - alpha, axis=0)
    t_before = np.concatenate([np.ones((1, alpha.shape[1])), t_after[:-1]], axis=0)
    contrib = t_before >= stop
    w = alpha * t_before * contrib
    last = contrib.sum(axis=0) - 1
    t_final = np.where(last >= 0, t_after[np.maximum(last, 0), np.arange(alpha.shape[1])], 1.0)
    return t_before, contrib, w, t_final


def render(cloud, K, T, height, width, cfg, tile_rows=None, prepared=None, margins=False):
    """Colour/depth/feature/alpha + per-pixel live-contributor counts.

    tile_rows: optional iterable of tile-row indices to composite (used by the
    bounded CPU baseline); other pixels stay at background.
    prepared: optional (proj, lists) from project()/bin_tiles() to reuse.
    margins: also return the per-pixel decision margins (pixel_decision_margins)
    computed in the same tile loop (out["margins"])."""
    if prepared is None:
        proj = project(cloud, K, T, height, width, cfg)
        lists = bin_tiles(proj, height, width, cfg.tile)
    else:
        proj, lists = prepared
    tile = cfg.tile
    n = proj["feature"].shape[1]
    color = np.zeros((height, width, 3))
    depth = np.zeros((height, width))
    feature = np.zeros((height, width, n))
    tfin = np.ones((height, width))
    ncontrib = np.zeros((height, width), dtype=np.int64)
    margin_a = np.full((height, width), np.inf) if margins else None
    margin_s = np.full((height, width), np.inf) if margins else None
    tiles = {}
    rows_to_do = range(len(lists)) if tile_rows is None else tile_rows
    for ty in rows_to_do:
        ys = np.arange(ty * tile, min(ty * tile + tile, height))
        for tx, rows in enumerate(lists[ty]):
            if rows.size == 0:
                continue
            xs = np.arange(tx * tile, min(tx * tile + tile, width))
            alpha, g, a_raw, dx, dy, q, inside = tile_alpha(proj, rows, xs, ys, cfg)
            t_before, contrib, w, t_final = transmittance(alpha, cfg.stop_transmittance)
            shp = (ys.size, xs.size)
            if margins:
                a_m, s_m = _tile_margins(alpha, a_raw, q, inside, t_before, cfg, proj["opacity"][rows])
                margin_a[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1] = a_m.min(axis=0).reshape(shp)
                margin_s[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1] = s_m.min(axis=0).reshape(shp)
            sl = (slice(ys[0], ys[-1] + 1), slice(xs[0], xs[-1] + 1))
            color[sl] = (w.T @ proj["color"][rows]).reshape(shp + (3,))
            depth[sl] = (w.T @ proj["view_depth"][rows]).reshape(shp)
            if n:
                feature[sl] = (w.T @ proj["feature"][rows]).reshape(shp + (n,))
            tfin[sl] = t_final.reshape(shp)
            ncontrib[sl] = (contrib & (alpha > 0)).sum(axis=0).reshape(shp)
            tiles[(ty, tx)] = (rows, xs, ys)
    color = color + tfin[:, :, None] * cfg.background[None, None, :]
    out = {"color": color, "depth": depth, "feature": feature, "alpha": 1.0 - tfin,
           "n_contrib": ncontrib, "proj": proj, "tiles": tiles, "t_final": tfin}
    if margins:
        out["alpha_margins"], out["stop_margins"] = margin_a, margin_s
        out["margins"] = np.minimum(margin_a, margin_s)
    return out


# ---------------------------------------------------------------------------
# backward (rasterizer.py:320-452)
# ---------------------------------------------------------------------------
def render_backward(cloud, K, T, height, width, cfg, out, d_color=None, d_depth=None,
                    d_feature=None, d_alpha=None):
    proj = out["proj"]
    m = proj["source_index"].size
    n = proj["feature"].shape[1]
    z2 = lambda *s: np.zeros(s)  # noqa: E731
    dC = z2(height, width, 3) if d_color is None else np.asarray(d_color, dtype=np.float64)
    dD = z2(height, width) if d_depth is None else np.asarray(d_depth, dtype=np.float64)
    dF = z2(height, width, n) if d_feature is None else np.asarray(d_feature, dtype=np.float64)
    dA = z2(height, width) if d_alpha is None else np.asarray(d_alpha, dtype=np.float64)
    g_op = np.zeros(m)
    g_col = np.zeros((m, 3))
    g_feat = np.zeros((m, n))
    g_z = np.zeros(m)
    g_mean = np.zeros((m, 2))
    g_con = np.zeros((m, 2, 2))
    for (ty, tx), (rows, xs, ys) in out["tiles"].items():
        alpha, g, a_raw, dx, dy, q, inside = tile_alpha(proj, rows, xs, ys, cfg)
        t_before, contrib, w, t_final = transmittance(alpha, cfg.stop_transmittance)
        sl = (slice(ys[0], ys[-1] + 1), slice(xs[0], xs[-1] + 1))
        P = ys.size * xs.size
        uc, ud, uf, ua = dC[sl].reshape(P, 3), dD[sl].reshape(P), dF[sl].reshape(P, n), dA[sl].reshape(P)
        g_col[rows] += w @ uc
        g_z[rows] += w @ ud
        if n:
            g_feat[rows] += w @ uf
        uval = proj["color"][rows] @ uc.T + proj["view_depth"][rows][:, None] * ud[None, :]
        if n:
            uval = uval + proj["feature"][rows] @ uf.T
        vpix = uc @ cfg.background - ua
        wu = w * uval
        behind = np.cumsum(wu[::-1], axis=0)[::-1] - wu
        live = contrib & (alpha > 0)
        safe = np.where(live, 1.0 - alpha, 1.0)
        dal = np.where(live, uval * t_before - (behind + t_final[None, :] * vpix[None, :]) / safe, 0.0)
        dar = dal * (a_raw < cfg.alpha_cap)
        g_op[rows] += (dar * g).sum(axis=1)
        dq = -0.5 * g * dar * proj["opacity"][rows][:, None]
        sxx, sxy, syy = (dq * dx * dx).sum(1), (dq * dx * dy).sum(1), (dq * dy * dy).sum(1)
        g_con[rows, 0, 0] += sxx
        g_con[rows, 0, 1] += sxy
        g_con[rows, 1, 0] += sxy
        g_con[rows, 1, 1] += syy
        con = proj["conic"][rows]
        g_mean[rows, 0] -= 2.0 * (dq * (con[:, 0, 0, None] * dx + con[:, 0, 1, None] * dy)).sum(1)
        g_mean[rows, 1] -= 2.0 * (dq * (con[:, 1, 0, None] * dx + con[:, 1, 1, None] * dy)).sum(1)

    C = proj["conic"]
    g_cov2 = -C @ g_con @ C
    K = np.asarray(K, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    R, tv = T[:3, :3], T[:3, 3]
    fx, fy = K[0, 0], K[1, 1]
    src = proj["source_index"]
    pos = np.asarray(cloud.positions, dtype=np.float64)[src]
    cam = pos @ R.T + tv
    x, y, z = cam[:, 0], cam[:, 1], cam[:, 2]
    quats = np.asarray(cloud.rotations, dtype=np.float64)[src]
    lsc = np.asarray(cloud.log_scales, dtype=np.float64)[src]
    sig = covariances(quats, lsc)
    J = np.zeros((m, 2, 3))
    J[:, 0, 0], J[:, 0, 2] = fx / z, -fx * x / (z * z)
    J[:, 1, 1], J[:, 1, 2] = fy / z, -fy * y / (z * z)
    M = J @ R
    g_M = (g_cov2 + np.transpose(g_cov2, (0, 2, 1))) @ M @ sig
    g_sig = np.transpose(M, (0, 2, 1)) @ g_cov2 @ M
    g_J = g_M @ R.T
    g_cam = np.zeros((m, 3))
    g_cam[:, 0] = g_J[:, 0, 2] * (-fx / z ** 2) + g_mean[:, 0] * fx / z
    g_cam[:, 1] = g_J[:, 1, 2] * (-fy / z ** 2) + g_mean[:, 1] * fy / z
    g_cam[:, 2] = (g_J[:, 0, 0] * (-fx / z ** 2) + g_J[:, 0, 2] * (2 * fx * x / z ** 3)
                   + g_J[:, 1, 1] * (-fy / z ** 2) + g_J[:, 1, 2] * (2 * fy * y / z ** 3)
                   - g_mean[:, 0] * fx * x / z ** 2 - g_mean[:, 1] * fy * y / z ** 2 + g_z)
    g_pos = g_cam @ R
    g_q, g_ls = covariance_grads(quats, lsc, g_sig)
    o = proj["opacity"]
    raw = proj["color_raw"]
    gate = (raw > 0.0) & (raw < 1.0)
    g_colg = g_col * gate
    k = len(np.asarray(cloud.positions))
    out_g = {
        "positions": np.zeros((k, 3)), "rotations": np.zeros((k, 4)), "log_scales": np.zeros((k, 3)),
        "opacity_logits": np.zeros(k), "colors_raw": np.zeros((k, 3)),
        "features": np.zeros((k, np.shape(cloud.features)[1])),
        "viewspace_index": src.copy(),
        "viewspace_norm": np.hypot(g_mean[:, 0] * 0.5 * width, g_mean[:, 1] * 0.5 * height),
    }
    deg = sh_degree_of(cloud)
    if deg > 0:
        d, dn = view_dirs(pos, T)
        Y = sh_basis(deg, d)
        sh = np.asarray(cloud.sh_rest, dtype=np.float64)[src]
        gsh = np.zeros((k,) + np.shape(cloud.sh_rest)[1:])
        gsh[src] = Y[:, :, None] * g_colg[:, None, :]
        out_g["sh_rest"] = gsh
        # through the view direction: numerical Jacobian of the basis (oracle side)
        eps = 1e-6
        gdir = np.zeros((m, 3))
        w_c = np.einsum("nkc,nc->nk", sh, g_colg)
        for ax in range(3):
            dp = d.copy()
            dp[:, ax] += eps
            dm = d.copy()
            dm[:, ax] -= eps
            gdir[:, ax] = ((sh_basis(deg, dp) - sh_basis(deg, dm)) / (2 * eps) * w_c).sum(1)
        g_pos = g_pos + (gdir - (gdir * d).sum(1, keepdims=True) * d) / dn[:, None]
    out_g["positions"][src] = g_pos
    out_g["rotations"][src] = g_q
    out_g["log_scales"][src] = g_ls
    out_g["opacity_logits"][src] = g_op * o * (1.0 - o)
    out_g["colors_raw"][src] = g_colg
    if n:
        out_g["features"][src, :n] = g_feat
    return out_g


# ---------------------------------------------------------------------------
# HexPlane (hexplane.py:84-187)
# ---------------------------------------------------------------------------
def field_coords(aabb, positions, t):
    lo, hi = aabb[0], aabb[1]
    raw = (positions - lo) / (hi - lo)
    inside = (raw > 0.0) & (raw < 1.0)
    c = np.empty((positions.shape[0], 4))
    c[:, :3] = np.clip(raw, 0.0, 1.0)
    c[:, 3] = np.clip(t, 0.0, 1.0)
    return c, inside


def _cell(res_a, res_b, ca, cb):
    u, v = ca * (res_a - 1), cb * (res_b - 1)
    i0 = np.clip(np.floor(u).astype(np.int64), 0, res_a - 2)
    j0 = np.clip(np.floor(v).astype(np.int64), 0, res_b - 2)
    return i0, j0, u - i0, v - j0


def _lerp4(plane, i0, j0, fa, fb):
    fa, fb = fa[:, None], fb[:, None]
    c00, c10 = plane[i0, j0], plane[i0 + 1, j0]
    c01, c11 = plane[i0, j0 + 1], plane[i0 + 1, j0 + 1]
    val = (1 - fa) * (1 - fb) * c00 + fa * (1 - fb) * c10 + (1 - fa) * fb * c01 + fa * fb * c11
    return val, (c00, c10, c01, c11)


def hexplane_query(planes, aabb, positions, t):
    """Latent [K, C*levels]: per level the left-to-right product of six
    bilinear samples, levels concatenated (hexplane.py:118-142)."""
    c, _ = field_coords(np.asarray(aabb, dtype=np.float64), np.asarray(positions, dtype=np.float64), t)
    out = []
    for level in planes:
        acc = None
        for plane, (a0, a1) in zip(level, PLANE_AXES):
            plane = np.asarray(plane, dtype=np.float64)
            i0, j0, fa, fb = _cell(plane.shape[0], plane.shape[1], c[:, a0], c[:, a1])
            s, _ = _lerp4(plane, i0, j0, fa, fb)
            acc = s if acc is None else acc * s
        out.append(acc)
    return np.concatenate(out, axis=1)


def hexplane_backward(planes, aabb, positions, t, d_latent):
    """Plane gradients (scatter-add) and position gradients (hexplane.py:145-187)."""
    aabb = np.asarray(aabb, dtype=np.float64)
    positions = np.asarray(positions, dtype=np.float64)
    c, inside = field_coords(aabb, positions, t)
    k = positions.shape[0]
    dco = np.zeros((k, 4))
    grads = []
    off = 0
    for level in planes:
        C = np.shape(level[0])[2]
        up = d_latent[:, off:off + C]
        off += C
        samples, parts = [], []
        for plane, (a0, a1) in zip(level, PLANE_AXES):
            plane = np.asarray(plane, dtype=np.float64)
            i0, j0, fa, fb = _cell(plane.shape[0], plane.shape[1], c[:, a0], c[:, a1])
            s, corners = _lerp4(plane, i0, j0, fa, fb)
            samples.append(s)
            parts.append((i0, j0, fa, fb, corners))
        lvl = []
        for p, (plane, (a0, a1)) in enumerate(zip(level, PLANE_AXES)):
            others = np.ones_like(up)
            for q, s in enumerate(samples):
                if q != p:
                    others = others * s
            coef = up * others
            i0, j0, fa, fb, (c00, c10, c01, c11) = parts[p]
            ra, rb = np.shape(plane)[:2]
            gp = np.zeros((ra, rb, C))
            for di, dj, wgt in ((0, 0, (1 - fa) * (1 - fb)), (1, 0, fa * (1 - fb)),
                                (0, 1, (1 - fa) * fb), (1, 1, fa * fb)):
                np.add.at(gp, (i0 + di, j0 + dj), coef * wgt[:, None])
            lvl.append(gp)
            fa2, fb2 = fa[:, None], fb[:, None]
            dco[:, a0] += (coef * ((1 - fb2) * (c10 - c00) + fb2 * (c11 - c01))).sum(1) * (ra - 1)
            dco[:, a1] += (coef * ((1 - fa2) * (c01 - c00) + fa2 * (c11 - c10))).sum(1) * (rb - 1)
        grads.append(lvl)
    dpos = dco[:, :3] / (aabb[1] - aabb[0]) * inside
    return grads, dpos


# ---------------------------------------------------------------------------
# MLP + deformation (numerics.py:56-105, deformation.py:100-183)
# ---------------------------------------------------------------------------
def dense_stack(layers, x):
    """layers: list of (W [out,in], b [out], relu).  Returns output and the
    per-layer (input, pre-activation) record (numerics.py:56-75)."""
    h = x
    rec = []
    for W, b, relu in layers:
        pre = h @ np.asarray(W, dtype=np.float64).T + np.asarray(b, dtype=np.float64)
        rec.append((h, pre))
        h = np.maximum(pre, 0.0) if relu else pre
    return h, rec


def dense_stack_backward(layers, rec, gy):
    """numerics.py:78-105: returns (dx, [(dW, db), ...])."""
    g = gy
    out = [None] * len(layers)
    for i in range(len(layers) - 1, -1, -1):
        W, _, relu = layers[i]
        x_in, pre = rec[i]
        if relu:
            g = g * (pre > 0.0)
        out[i] = (g.T @ x_in, g.sum(axis=0))
        g = g @ np.asarray(W, dtype=np.float64)
    return g, out


def deform(cloud, planes, aabb, net, t, enable_grid=True, enable_feature_update=True):
    """net: dict stack-name -> list of (W, b, relu) with names of
    DeformationNet.stacks() (deformation.py:61-66).  Returns (snapshot dict, cache)."""
    pos = np.asarray(cloud.positions, dtype=np.float64)
    k = pos.shape[0]
    latent_dim = np.shape(net["net.trunk"][0][0])[1]
    lat = hexplane_query(planes, aabb, pos, t) if enable_grid else np.zeros((k, latent_dim))
    hid, trunk_rec = dense_stack(net["net.trunk"], lat)
    deltas, e2s, recs = {}, {}, {}
    for name in BRANCHES:
        e2, erec = dense_stack(net[f"net.ext.{name}"], hid)
        d, hrec = dense_stack(net[f"net.head.{name}"], e2)
        deltas[name], e2s[name], recs[name] = d, e2, (erec, hrec)
    feats = np.asarray(cloud.features, dtype=np.float64)
    frec = None
    if enable_feature_update:
        dz, frec = dense_stack(net["net.feat"], np.concatenate([e2s[b] for b in BRANCHES], axis=1))
        feats = feats + dz
    snap = {
        "positions": pos + deltas["position"],
        "rotations": np.asarray(cloud.rotations, dtype=np.float64) + deltas["rotation"],
        "log_scales": np.asarray(cloud.log_scales, dtype=np.float64) + deltas["scale"],
        "opacity_logits": np.asarray(cloud.opacity_logits, dtype=np.float64) + deltas["opacity"][:, 0],
        "colors_raw": np.asarray(cloud.colors_raw, dtype=np.float64),
        "features": feats,
    }
    cache = {"trunk": trunk_rec, "branch": recs, "feat": frec, "t": t}
    return snap, cache


def relu_gate_margins(net, cache):
    """Per Gaussian, the smallest relative margin of any ReLU gate
    (numerics.py:72, 99: pre > 0) in the deformation MLP:
    |pre| / (sum_i |W_oi x_i| + |b_o|).  A gate inside the device's
    product-rounding band (tensor-core bf16x3 operands carry ~2^-17 relative
    error) may resolve either way; its Gaussian is 'ambiguous' under the
    parity contract."""
    def stack(layers, rec, m):
        for (W, b, relu), (x, pre) in zip(layers, rec):
            if not relu:
                continue
            scale = np.abs(x) @ np.abs(np.asarray(W, dtype=np.float64)).T + np.abs(np.asarray(b, dtype=np.float64))
            m = np.minimum(m, (np.abs(pre) / np.maximum(scale, 1e-300)).min(axis=1))
        return m

    k = cache["trunk"][0][0].shape[0]
    m = stack(net["net.trunk"], cache["trunk"], np.full(k, np.inf))
    for name in BRANCHES:
        erec, hrec = cache["branch"][name]
        m = stack(net[f"net.ext.{name}"], erec, m)
        m = stack(net[f"net.head.{name}"], hrec, m)
    if cache["feat"] is not None:
        m = stack(net["net.feat"], cache["feat"], m)
    return m


def deform_backward(cloud, planes, aabb, net, cache, grads, enable_grid=True,
                    enable_feature_update=True):
    """deformation.py:139-183.  grads: dict with positions, rotations,
    log_scales, opacity_logits, features.  Returns (cloud_grads, net_grads, plane_grads)."""
    k = np.shape(cloud.positions)[0]
    half = np.shape(net["net.ext.position"][0][0])[0]
    net_grads = {}

    def put(prefix, gl):
        for i, (dw, db) in enumerate(gl):
            net_grads[f"{prefix}.{i}.weight"] = dw
            net_grads[f"{prefix}.{i}.bias"] = db

    d_e2 = {b: np.zeros((k, half)) for b in BRANCHES}
    if enable_feature_update:
        dj, fg = dense_stack_backward(net["net.feat"], cache["feat"], np.asarray(grads["features"]))
        put("net.feat", fg)
        for i, b in enumerate(BRANCHES):
            d_e2[b] = d_e2[b] + dj[:, i * half:(i + 1) * half]
    up = {"position": grads["positions"], "rotation": grads["rotations"],
          "scale": grads["log_scales"], "opacity": np.asarray(grads["opacity_logits"])[:, None]}
    d_hid = 0.0
    for b in BRANCHES:
        erec, hrec = cache["branch"][b]
        dg, hg = dense_stack_backward(net[f"net.head.{b}"], hrec, np.asarray(up[b], dtype=np.float64))
        put(f"net.head.{b}", hg)
        dh, eg = dense_stack_backward(net[f"net.ext.{b}"], erec, dg + d_e2[b])
        put(f"net.ext.{b}", eg)
        d_hid = d_hid + dh
    d_lat, tg = dense_stack_backward(net["net.trunk"], cache["trunk"], d_hid)
    put("net.trunk", tg)
    cg = {"positions": np.array(grads["positions"], dtype=np.float64)}
    pg = None
    if enable_grid:
        pg, dpos = hexplane_backward(planes, aabb, cloud.positions, cache["t"], d_lat)
        cg["positions"] = cg["positions"] + dpos
    return cg, net_grads, pg


# ---------------------------------------------------------------------------
# margins for the discrete parity contract
# ---------------------------------------------------------------------------
def projection_margins(proj, height, width, tile, cfg):
    """Relative distance of every discrete projection/binning decision of the
    *kept* Gaussians to its flip point: ceil argument vs integer, (u±r)/tile
    vs integer, offscreen inequalities, and the relative depth gap to the
    depth-order neighbours (exact ties resolve by source index on both sides
    and are not ambiguous).  The device evaluates these in fp64, so callers
    compare them against an fp64-level threshold."""
    u, v, r = proj["mean2d"][:, 0], proj["mean2d"][:, 1], proj["radius"]
    src = proj["source_index"]
    pos_in_front = np.searchsorted(proj["front_index"], src)
    arg = proj["front_radius_arg"][pos_in_front]
    m = np.abs(arg - np.round(arg)) / np.maximum(np.abs(arg), 1.0)
    for e in ((u - r) / tile, (u + r) / tile, (v - r) / tile, (v + r) / tile):
        m = np.minimum(m, np.abs(e - np.round(e)) / np.maximum(np.abs(e), 1.0))
    for e in (u + r, (width - 1) - (u - r), v + r, (height - 1) - (v - r)):
        m = np.minimum(m, np.abs(e) / np.maximum(np.abs(u) + r + width, 1.0))
    # pixel footprint bounds: |j - u| <= r decided per integer column/row
    for e in (u - r, u + r, v - r, v + r):
        m = np.minimum(m, np.abs(e - np.round(e)) / np.maximum(np.abs(e), 1.0))
    z = proj["view_depth"]
    if z.size > 1:
        gap = np.abs(np.diff(z)) / np.maximum(np.abs(z[1:]), 1e-12)
        gap = np.where(gap == 0.0, np.inf, gap)
        gl = np.concatenate([[np.inf], gap])
        gr = np.concatenate([gap, [np.inf]])
        m = np.minimum(m, np.minimum(gl, gr))
    return m


def _tile_margins(alpha, a_raw, q, inside, t_before, cfg, opac):
    """[G, P] relative margins of one tile's fp32 blend decisions (see
    pixel_decision_margins), split into (per-Gaussian alpha decisions:
    q-skip, alpha-skip, alpha-cap; the stop rule |T_after - stop| / stop);
    rows the traversal cannot reach are inf.  The q-skip test only decides
    anything for opacities within 1e-4 of 1: at q = 2 ln 255 the raw alpha is
    opacity/255, below the alpha-skip threshold either way."""
    reach = t_before >= cfg.stop_transmittance * 0.5  # rows the traversal can see
    q_matters = (opac * np.exp(-0.5 * Q_SKIP) >= cfg.alpha_skip * (1.0 - 1e-4))[:, None]
    mm = np.where((inside | (q > Q_SKIP)) & q_matters, np.abs(q - Q_SKIP) / Q_SKIP, np.inf)
    am = np.minimum(a_raw, cfg.alpha_cap)
    mm = np.minimum(mm, np.where(inside, np.abs(am - cfg.alpha_skip) / cfg.alpha_skip, np.inf))
    mm = np.minimum(mm, np.where(inside, np.abs(a_raw - cfg.alpha_cap) / cfg.alpha_cap, np.inf))
    t_after = t_before * (1.0 - alpha)
    ms = np.where(alpha > 0, np.abs(t_after - cfg.stop_transmittance) / cfg.stop_transmittance, np.inf)
    return np.where(reach, mm, np.inf), np.where(reach, ms, np.inf)


def pixel_decision_margins(out, cfg, split=False):
    """Per pixel: the smallest relative margin of any fp32-evaluated blend
    decision met while compositing it (alpha-skip, alpha-cap, q-skip, stop).
    The square-footprint test is decided from fp64 integer bounds on device
    and is covered by projection_margins.  split=True returns (alpha
    decisions, stop rule) separately: the stop rule compares a transmittance
    that is a product over every earlier contributor, so its fp32 error grows
    with the contributor count and callers may give it its own threshold.
    render(..., margins=True) computes the same arrays in its own tile loop."""
    if "margins" in out:
        return (out["alpha_margins"], out["stop_margins"]) if split else out["margins"]
    proj = out["proj"]
    h, w = out["t_final"].shape
    ma = np.full((h, w), np.inf)
    ms = np.full((h, w), np.inf)
    for (ty, tx), (rows, xs, ys) in out["tiles"].items():
        alpha, g, a_raw, dx, dy, q, inside = tile_alpha(proj, rows, xs, ys, cfg)
        t_before, contrib, wts, t_final = transmittance(alpha, cfg.stop_transmittance)
        a_m, s_m = _tile_margins(alpha, a_raw, q, inside, t_before, cfg, proj["opacity"][rows])
        sl = (slice(ys[0], ys[-1] + 1), slice(xs[0], xs[-1] + 1))
        if rows.size:
            ma[sl] = a_m.min(axis=0).reshape(ys.size, xs.size)
            ms[sl] = s_m.min(axis=0).reshape(ys.size, xs.size)
    return (ma, ms) if split else np.minimum(ma, ms)


def reached_rows(out, cfg, pixels, stop_pixels=None):
    """Projected rows (bool [M]) whose backward sums include a term that an
    ambiguous decision can change.  `pixels` (bool [H, W]): pixels with an
    ambiguous alpha decision -- every Gaussian the traversal reaches there
    with a non-zero or near-threshold alpha (a flipped alpha rescales the
    transmittance of everything behind it).  `stop_pixels`: pixels whose only
    ambiguity is the stop rule -- the flip adds or drops a contributor of
    weight ~alpha * 1e-4, which moves the earlier contributors' terms there
    by ~1e-4 relative, so only the Gaussians near the stop (T_before within
    [stop/2, 2 stop]) are marked."""
    proj = out["proj"]
    hit = np.zeros(proj["source_index"].size, dtype=bool)
    stop = cfg.stop_transmittance
    sp = np.zeros_like(pixels) if stop_pixels is None else stop_pixels
    for (ty, tx), (rows, xs, ys) in out["tiles"].items():
        sub = pixels[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1].reshape(-1)
        ssub = sp[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1].reshape(-1)
        if rows.size == 0 or not (sub.any() or ssub.any()):
            continue
        alpha, g, a_raw, dx, dy, q, inside = tile_alpha(proj, rows, xs, ys, cfg)
        t_before, _, _, _ = transmittance(alpha, stop)
        near = inside | (q <= Q_SKIP * 1.01)
        reach = (t_before >= stop * 0.5) & near
        tail = reach & (t_before <= stop * 2.0)
        hit[rows[reach[:, sub].any(axis=1) | tail[:, ssub].any(axis=1)]] = True
    return hit


# ---------------------------------------------------------------------------
# training-step glue
# ---------------------------------------------------------------------------
def adam_update(param, grad, m, v, step_count, lr, eps, beta1=0.9, beta2=0.999):
    """numerics.py:137-159: returns (new_param, new_m, new_v, new_step_count);
    raises OracleError('numeric') on a non-finite gradient before touching
    anything, 'config' on a non-positive learning rate."""
    if not lr > 0.0:
        raise OracleError("config", f"learning rate must be positive, got {lr}")
    grad = np.asarray(grad, dtype=np.float64)
    if not np.all(np.isfinite(grad)):
        raise OracleError("numeric", f"non-finite gradient ({int(np.sum(~np.isfinite(grad)))}/{grad.size} entries)")
    step = step_count + 1
    m_new = beta1 * m + (1.0 - beta1) * grad
    v_new = beta2 * v + (1.0 - beta2) * grad * grad
    corr_m = m_new / (1.0 - beta1 ** step)
    corr_v = v_new / (1.0 - beta2 ** step)
    return param - lr * corr_m / (np.sqrt(corr_v) + eps), m_new, v_new, step


def learning_rate(lr_init, lr_final, max_steps, t, delay_mult=1.0, delay_steps=0):
    """numerics.py:189-199 (log-linear interpolation + optional sine ramp)."""
    frac = min(t, max_steps) / max_steps
    lr = np.exp((1.0 - frac) * np.log(lr_init) + frac * np.log(lr_final)) if lr_init != lr_final else lr_init
    if delay_steps > 0:
        ramp = min(max(t / delay_steps, 0.0), 1.0)
        lr = lr * (delay_mult + (1.0 - delay_mult) * np.sin(0.5 * np.pi * ramp))
    return float(lr)


def total_variation(planes, scale=1.0):
    """hexplane.py:190-222: (sum over planes of mean squared axis-adjacent
    differences, d(scale*tv)/d(plane) per plane)."""
    total = 0.0
    grads = []
    for level in planes:
        lg = []
        for p in level:
            p = np.asarray(p, dtype=np.float64)
            ra, rb, c = p.shape
            n = ((ra - 1) * rb + ra * (rb - 1)) * c
            fa = np.diff(p, axis=0)  # p[a+1]-p[a]
            fb = np.diff(p, axis=1)
            total += (np.sum(fa ** 2) + np.sum(fb ** 2)) / n
            g = np.zeros_like(p)
            k = 2.0 * scale / n
            g[1:] += k * fa
            g[:-1] -= k * fa
            g[:, 1:] += k * fb
            g[:, :-1] -= k * fb
            lg.append(g)
        grads.append(lg)
    return total, grads


def _resize_axis(n_in, n_out):
    """semantic.py:82-90: corner-aligned source index and weight per output."""
    pos = np.full(1, 0.5 * (n_in - 1)) if n_out == 1 else np.arange(n_out) * (n_in - 1) / (n_out - 1)
    lo = np.clip(np.floor(pos).astype(np.int64), 0, max(n_in - 2, 0))
    return lo, np.minimum(lo + 1, n_in - 1), pos - lo


def resize_matrix(n_in, n_out):
    """Dense [n_out, n_in] interpolation matrix of one axis (so resize and
    its adjoint are A·X·Bᵀ and Aᵀ·G·B — an independent restatement of
    semantic.py:93-123)."""
    lo, hi, f = _resize_axis(n_in, n_out)
    A = np.zeros((n_out, n_in))
    np.add.at(A, (np.arange(n_out), lo), 1.0 - f)
    np.add.at(A, (np.arange(n_out), hi), f)
    return A


def resize(img, out_hw):
    img = np.asarray(img, dtype=np.float64)
    Ay = resize_matrix(img.shape[0], out_hw[0])
    Ax = resize_matrix(img.shape[1], out_hw[1])
    return np.einsum("yi,ijc,xj->yxc", Ay, img, Ax)


def resize_adjoint(d_out, in_hw):
    d_out = np.asarray(d_out, dtype=np.float64)
    Ay = resize_matrix(in_hw[0], d_out.shape[0])
    Ax = resize_matrix(in_hw[1], d_out.shape[1])
    return np.einsum("yi,yxc,xj->ijc", Ay, d_out, Ax)


def decoder_forward(weight, bias, rendered, out_hw):
    """semantic.py:150-158."""
    r = resize(rendered, out_hw)
    return r @ np.asarray(weight).T + bias, r


def decoder_backward(weight, resized, in_hw, d_out):
    """semantic.py:161-168: (d_rendered, d_weight, d_bias)."""
    d_out = np.asarray(d_out, dtype=np.float64)
    d_bias = d_out.reshape(-1, d_out.shape[2]).sum(axis=0)
    d_weight = d_out.reshape(-1, d_out.shape[2]).T @ resized.reshape(-1, resized.shape[2])
    return resize_adjoint(d_out @ np.asarray(weight), in_hw), d_weight, d_bias


def l1_mean_pixels(pred, gt):
    """semantic.py:171-181: (sum|pred-gt|/(H*W), sign(pred-gt)/(H*W))."""
    d = np.asarray(pred, dtype=np.float64) - np.asarray(gt, dtype=np.float64)
    hw = d.shape[0] * d.shape[1]
    return float(np.abs(d).sum() / hw), np.sign(d) / hw


def photometric(color, image, mask, depth, depth_target, alpha, lambda_rgb=1.0, lambda_depth=1.0):
    """training.py:300-338: (rgb, depth_term, dC, dD) with dmask = mask & alpha>=0.5."""
    mask = np.ones(color.shape[:2], bool) if mask is None else np.asarray(mask, bool)
    n_rgb = 3 * int(mask.sum())
    diff = np.asarray(color, np.float64) - image
    rgb = float(np.abs(diff)[mask].sum() / n_rgb) if n_rgb else 0.0
    dC = lambda_rgb * np.sign(diff) * mask[:, :, None] / n_rgb if n_rgb else np.zeros_like(diff)
    if depth is None:
        return rgb, 0.0, dC, None
    dmask = mask & (np.asarray(alpha) >= 0.5)
    n_d = int(dmask.sum())
    dd = np.asarray(depth, np.float64) - depth_target
    dterm = float(np.abs(dd)[dmask].sum() / n_d) if n_d else 0.0
    dD = lambda_depth * np.sign(dd) * dmask / n_d if n_d else np.zeros_like(dd)
    return rgb, dterm, dC, dD


def density_control(cloud, accum, count, grad_threshold, percent_dense, prune_opacity, split_factor, extent,
                    normals=None, prune_only=False, extras=()):
    """gaussians.py:349-417 restated: returns (new arrays dict, new accum, new
    count, new extras, counts dict).  normals: [2, n_split, 3] samples (the
    reference draws rng.standard_normal((n_split, 3)) twice)."""
    fields = ["positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features"]
    if getattr(cloud, "sh_rest", None) is not None:
        fields.append("sh_rest")
    arrs = {f: np.asarray(getattr(cloud, f), dtype=np.float64) for f in fields}
    prune = sigmoid(arrs["opacity_logits"]) < prune_opacity
    k = len(prune)
    if prune_only:
        keep = ~prune
        out = {f: a[keep] for f, a in arrs.items()}
        return out, accum[keep], count[keep], [e[keep] for e in extras], {"keep": int(keep.sum())}
    avg = accum / np.maximum(count, 1.0)
    high = avg >= grad_threshold
    small = np.exp(arrs["log_scales"]).max(axis=1) <= percent_dense * extent
    clone = high & small & ~prune
    split = high & ~small & ~prune
    keep = ~(prune | (high & ~small))
    ci, si = np.nonzero(clone)[0], np.nonzero(split)[0]
    parts = {f: [a[keep], a[ci]] for f, a in arrs.items()}
    if si.size:
        q = arrs["rotations"][si]
        q = q / np.linalg.norm(q, axis=1, keepdims=True)
        R = rotation_from_unit_quats(q)
        s = np.exp(arrs["log_scales"][si])
        for j in range(2):
            off = np.einsum("kij,kj->ki", R, normals[j] * s)
            for f, a in arrs.items():
                rows = a[si].copy()
                if f == "positions":
                    rows = rows + off
                elif f == "log_scales":
                    rows = rows - np.log(split_factor)
                parts[f].append(rows)
    out = {f: np.concatenate(p, axis=0) for f, p in parts.items()}
    n_new = len(out["positions"]) - int(keep.sum())
    new_extras = [np.concatenate([e[keep], np.zeros((n_new,) + e.shape[1:])]) for e in extras]
    n = len(out["positions"])
    return out, np.zeros(n), np.zeros(n), new_extras, {"keep": int(keep.sum()), "clone": int(ci.size),
                                                       "split": int(si.size), "pruned": int(prune.sum())}
