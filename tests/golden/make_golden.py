"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package `featsplat` from /root/reference/pkg/src
(read-only, unmodified), feeds it seeded fp32-representable inputs and
stores inputs + reference outputs as .npz fixtures next to this script.  The
GPU box has no /root/reference; tests read only these fixtures.
"""

import importlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    sys.path.insert(0, REF_SRC)
    mods = {}
    for m in ("gaussians", "rasterizer", "hexplane", "deformation", "numerics", "semantic", "training"):
        mods[m] = importlib.import_module(f"featsplat.{m}")
    return mods


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def cloud_arrays(rng, k, nf, op_range, depth_range, xy=0.9, ls_range=(0.08, 0.35)):
    """conftest.random_cloud-style inputs (tests/conftest.py:17-27), rounded to fp32."""
    pos = np.column_stack([rng.uniform(-xy, xy, k), rng.uniform(-xy, xy, k),
                           rng.uniform(*depth_range, k)])
    rot = rng.normal(size=(k, 4))
    ls = np.log(rng.uniform(*ls_range, size=(k, 3)))
    p = rng.uniform(*op_range, k)
    return dict(positions=f32(pos), rotations=f32(rot), log_scales=f32(ls),
                opacity_logits=f32(np.log(p) - np.log1p(-p)),
                colors_raw=f32(rng.uniform(0.1, 0.9, size=(k, 3))),
                features=f32(rng.normal(size=(k, nf))))


def make_cloud(ref, arrs):
    G = ref["gaussians"].GaussianCloud
    return G(**{k: v.copy() for k, v in arrs.items()})


def frame(ref, h, w, focal, T=None, time=0.0):
    CF = ref["gaussians"].CameraFrame
    return CF(K=np.array([[focal, 0, (w - 1) / 2], [0, focal, (h - 1) / 2], [0, 0, 1.0]]),
              T=np.eye(4) if T is None else T, time=time, image=np.zeros((h, w, 3)),
              depth=np.zeros((h, w)), mask=np.ones((h, w), dtype=bool))


def rigid(rng, max_deg=5.0, max_t=0.1):
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = np.deg2rad(rng.uniform(-max_deg, max_deg))
    Kx = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + np.sin(ang) * Kx + (1 - np.cos(ang)) * Kx @ Kx
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = rng.uniform(-max_t, max_t, 3)
    return T


def render_case(ref, name, seed, k, h, w, nf, focal, bg, rigid_T=False, op_range=(0.05, 0.98),
                depth_range=(2.2, 3.8), with_backward=True, ls_range=(0.08, 0.35)):
    R = ref["rasterizer"]
    rng = np.random.default_rng(seed)
    arrs = cloud_arrays(rng, k, nf, op_range, depth_range, ls_range=ls_range)
    T = rigid(rng) if rigid_T else np.eye(4)
    fr = frame(ref, h, w, focal, T)
    cfg = R.RasterConfig(background=np.asarray(bg, dtype=np.float64))
    cloud = make_cloud(ref, arrs)
    out = R.render(cloud, fr, cfg)
    proj = out.record.proj
    tiles = R.bin_tiles(proj, h, w, cfg.tile)
    ranges, rows = [], []
    for row in tiles:
        for cell in row:
            ranges.append((len(rows), len(rows) + cell.size))
            rows.extend(cell.tolist())
    ncontrib = np.zeros((h, w), dtype=np.int64)
    for tr in out.record.tiles:
        _, contrib, _, _ = R._composite_weights(tr.alpha, cfg.stop_transmittance)
        live = (contrib & (tr.alpha > 0)).sum(axis=0).reshape(tr.ys.size, tr.xs.size)
        ncontrib[tr.y0:tr.y0 + tr.ys.size, tr.x0:tr.x0 + tr.xs.size] = live
    data = dict(K=fr.K, T=fr.T, height=h, width=w, background=cfg.background,
                color=out.color, depth=out.depth, feature=out.feature, alpha=out.alpha,
                n_contrib=ncontrib, proj_mean2d=proj.mean2d, proj_radius=proj.radius,
                proj_source_index=proj.source_index, proj_view_depth=proj.view_depth,
                proj_conic=proj.conic, proj_cov2d=proj.cov2d, proj_color=proj.color,
                proj_opacity=proj.opacity,
                tile_ranges=np.asarray(ranges, dtype=np.int64).reshape(-1, 2),
                tile_rows=np.asarray(rows, dtype=np.int64))
    data.update({f"cloud_{k_}": v for k_, v in arrs.items()})
    if with_backward:
        ups = dict(color=f32(rng.normal(size=(h, w, 3))), depth=f32(rng.normal(size=(h, w)) * 0.3),
                   feature=f32(rng.normal(size=(h, w, nf)) * 0.5),
                   alpha=f32(rng.normal(size=(h, w)) * 0.5))
        g = R.render_backward(cloud, fr, out, ups["color"], ups["depth"], ups["feature"], ups["alpha"])
        data.update({f"up_{k_}": v for k_, v in ups.items()})
        for f in ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features",
                  "viewspace_index", "viewspace_norm"):
            data[f"grad_{f}"] = getattr(g, f)
    np.savez_compressed(os.path.join(OUT, f"render_{name}.npz"), **data)
    print("render", name, "M =", len(proj), "pairs =", len(rows))


def deform_case(ref, name, seed, k, nf, width, depth, levels, base, out_dim, randomize=True):
    H, D, G = ref["hexplane"], ref["deformation"], ref["gaussians"]
    rng = np.random.default_rng(seed)
    arrs = cloud_arrays(rng, k, nf, (0.15, 0.3), (2.2, 3.8))
    aabb = np.array([[-1.2, -1.2, 1.8], [1.2, 1.2, 4.2]])
    field = H.HexPlaneField(H.HexPlaneConfig(levels=levels, base_resolution=base, out_dim=out_dim), aabb, rng)
    net = D.DeformationNet(field.latent_dim, D.DeformationConfig(width=width, depth=depth, feature_dim=nf), rng)
    for li, level in enumerate(field.planes):
        for pi in range(len(level)):
            field.planes[li][pi] = f32(0.8 + rng.normal(size=level[pi].shape) * 0.3) if randomize \
                else f32(level[pi])
    for prefix, stack in net.stacks():
        for layer in stack:
            layer.weight = f32(rng.normal(size=layer.weight.shape) * 0.2)
            layer.bias = f32(rng.normal(size=layer.bias.shape) * 0.2)
    cloud = G.GaussianCloud(**{k_: v.copy() for k_, v in arrs.items()})
    t = 0.61
    snap, cache = D.deform_with_cache(cloud, field, net, t)
    ups = {n_: f32(rng.normal(size=np.shape(getattr(cloud, n_))))
           for n_ in ("positions", "rotations", "log_scales", "opacity_logits", "features")}

    class Gr:
        pass

    gr = Gr()
    for n_, v in ups.items():
        setattr(gr, n_, v)
    cg, ng, pg = D.deform_backward(cloud, field, net, cache, gr)
    data = {f"cloud_{k_}": v for k_, v in arrs.items()}
    data.update(aabb=aabb, t=t, width=width, depth=depth, levels=np.asarray(levels),
                base=np.asarray(base), out_dim=out_dim, feature_dim=nf)
    for li, level in enumerate(field.planes):
        for pi, pl in enumerate(level):
            data[f"plane_{li}_{pi}"] = pl
            data[f"gplane_{li}_{pi}"] = pg[li][pi]
    for prefix, stack in net.stacks():
        for i, layer in enumerate(stack):
            data[f"w:{prefix}.{i}"] = layer.weight
            data[f"b:{prefix}.{i}"] = layer.bias
    for k_, v in ng.items():
        data[f"g:{k_}"] = v
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        data[f"snap_{f}"] = getattr(snap, f)
        data[f"up_{f}"] = ups[f]
    data["cg_positions"] = cg["positions"]
    data["latent"] = H.query(field, cloud.positions, t)
    np.savez_compressed(os.path.join(OUT, f"deform_{name}.npz"), **data)
    print("deform", name)


def train_ops_case(ref, seed=21):
    """Adam (3 steps, both eps), LR schedules, HexPlane TV, bilinear resize
    and adjoint, pointwise decoder fwd/bwd, feature L1 and the masked
    photometric grads -- all from the reference's own functions."""
    Nm, H, S, T = ref["numerics"], ref["hexplane"], ref["semantic"], ref["training"]
    rng = np.random.default_rng(seed)
    data = {}
    # Adam: numerics.py:137-159, three consecutive steps
    for tag, eps in (("g", 1e-15), ("n", 1e-8)):
        p = f32(rng.normal(size=(37, 5)))
        st = Nm.AdamState.for_param(p, eps=eps)
        data[f"adam_{tag}_p0"] = p
        for i in range(3):
            gr = f32(rng.normal(size=p.shape) * (10.0 ** rng.uniform(-6, 1)))
            if i == 1:
                gr[0, 0] = 0.0
            data[f"adam_{tag}_g{i}"] = gr
            p = Nm.adam_step(p, gr, st, 1e-3 * (i + 1))
            data[f"adam_{tag}_p{i + 1}"] = p
            data[f"adam_{tag}_m{i + 1}"] = st.m
            data[f"adam_{tag}_v{i + 1}"] = st.v
    # schedules: numerics.py:189-199
    steps = np.array([0, 1, 7, 500, 14000, 20000, 30000])
    data["lr_steps"] = steps
    data["lr_decay"] = np.array([Nm.lr_at_step(Nm.LrSchedule(1.6e-4, 1.6e-6, 20000), int(t)) for t in steps])
    data["lr_delay"] = np.array([Nm.lr_at_step(Nm.LrSchedule(1.6e-3, 1.6e-4, 20000, 0.01, 500), int(t))
                                 for t in steps])
    # TV: hexplane.py:190-222
    field = H.HexPlaneField(H.HexPlaneConfig(levels=(1, 2), base_resolution=(6, 5, 4, 3), out_dim=8),
                            np.array([[-1.0, -1, -1], [1, 1, 1]]), rng)
    for li, level in enumerate(field.planes):
        for pi in range(len(level)):
            field.planes[li][pi] = f32(rng.normal(size=level[pi].shape))
            data[f"tv_plane_{li}_{pi}"] = field.planes[li][pi]
    data["tv_loss"] = H.tv_loss(field)
    tg = H.tv_backward(field, 0.37)
    for li, level in enumerate(tg):
        for pi, g in enumerate(level):
            data[f"tv_grad_{li}_{pi}"] = g
    # resize (semantic.py:93-123): down, up, ragged, single-row/column
    for i, (hin, win, hout, wout) in enumerate(((12, 16, 5, 7), (5, 7, 12, 17), (9, 1, 4, 3), (1, 6, 1, 1))):
        img = f32(rng.normal(size=(hin, win, 3)))
        dout = f32(rng.normal(size=(hout, wout, 3)))
        data[f"rs{i}_in"], data[f"rs{i}_dout"] = img, dout
        data[f"rs{i}_out"] = S.resize_bilinear(img, (hout, wout))
        data[f"rs{i}_din"] = S.resize_bilinear_backward(dout, (hin, win))
    # decoder + feature loss (semantic.py:126-181), rendered N=6 -> teacher Ct=10
    dec = S.PointwiseDecoder.create(10, 6, rng)
    dec.weight = f32(dec.weight)
    dec.bias = f32(rng.normal(size=10) * 0.1)
    rendered = f32(rng.normal(size=(20, 24, 6)))
    teacher = f32(rng.normal(size=(9, 11, 10)))
    out, cache = S.decode_features_with_cache(dec, rendered, teacher.shape[:2])
    d_dec = 0.7 * S.feature_loss_backward(out, teacher)
    dr, dw, db = S.decode_features_backward(dec, cache, d_dec)
    data.update(dec_w=dec.weight, dec_b=dec.bias, dec_rendered=rendered, dec_teacher=teacher, dec_out=out,
                dec_loss=S.feature_loss(out, teacher), dec_d_rendered=dr, dec_dw=dw, dec_db=db)
    # masked photometric terms (training.py:300-338)
    h, w = 14, 18

    class Out:
        pass

    class Fr:
        pass

    o, fr = Out(), Fr()
    o.color = f32(rng.uniform(size=(h, w, 3)))
    o.depth = f32(rng.uniform(1, 3, size=(h, w)))
    o.alpha = f32(rng.uniform(size=(h, w)))
    fr.image = f32(rng.uniform(size=(h, w, 3)))
    fr.depth = f32(rng.uniform(1, 3, size=(h, w)))
    fr.mask = rng.uniform(size=(h, w)) > 0.3

    class Cfg:
        lambda_rgb = 0.8
        lambda_depth = 0.3

    rgb, depth, dC, dD = T._photometric_grads(o, fr, Cfg)
    data.update(ph_color=o.color, ph_depth=o.depth, ph_alpha=o.alpha, ph_image=fr.image, ph_depth_t=fr.depth,
                ph_mask=fr.mask, ph_rgb=rgb, ph_dterm=depth, ph_dC=dC, ph_dD=dD)
    np.savez_compressed(os.path.join(OUT, "train_ops.npz"), **data)
    print("train_ops")


def density_case(ref, seed=31):
    """densify_and_prune (clone + split + prune, with Adam states), then
    prune_only and reset_opacity, from the reference itself.  The split
    samples are recorded by replaying the same seeded generator."""
    G, Nm = ref["gaussians"], ref["numerics"]
    rng = np.random.default_rng(seed)
    k, nf = 400, 5
    arrs = cloud_arrays(rng, k, nf, (0.001, 0.9), (2.2, 3.8), ls_range=(0.002, 0.2))
    cloud = G.GaussianCloud(**{k_: v.copy() for k_, v in arrs.items()})
    stats = G.ViewspaceGradStats.zeros(k)
    idx = rng.integers(0, k, size=1500)
    norms = f32(rng.exponential(3e-4, size=1500))
    for i0 in range(0, 1500, 300):  # renders: distinct indices per call
        ii, pos = np.unique(idx[i0:i0 + 300], return_index=True)
        stats.add(ii, norms[i0:i0 + 300][pos])
    data = {f"cloud_{k_}": v for k_, v in arrs.items()}
    data.update(stats_accum=stats.accum.copy(), stats_count=stats.count.copy())
    adam = {}
    for name, arr in cloud.param_arrays().items():
        st = Nm.AdamState.for_param(arr)
        st.m = f32(rng.normal(size=arr.shape))
        st.v = f32(rng.uniform(size=arr.shape))
        adam[name] = st
        data[f"adam_{name}_m"], data[f"adam_{name}_v"] = st.m, st.v
    cfg = G.DensityControlConfig(grad_threshold=2e-4, percent_dense=0.05, prune_opacity=0.02, split_factor=1.6)
    extent = 1.3
    seed2 = 77
    split_rng = np.random.default_rng(seed2)
    rep = G.densify_and_prune(cloud, stats, 5, cfg, extent, split_rng, adam_states=adam)
    data.update(cfg=np.array([cfg.grad_threshold, cfg.percent_dense, cfg.prune_opacity, cfg.split_factor, extent]),
                split_seed=seed2, report=np.array([rep["cloned"], rep["split"], rep["pruned"], rep["count"]]))
    for name, arr in cloud.param_arrays().items():
        data[f"out_{name}"] = arr
        data[f"out_adam_{name}_m"], data[f"out_adam_{name}_v"] = adam[name].m, adam[name].v
    data.update(out_accum=stats.accum, out_count=stats.count)
    # prune_only on the densified cloud with fresh stats, then reset_opacity
    stats2 = G.ViewspaceGradStats(accum=f32(rng.uniform(size=len(cloud))), count=np.floor(rng.uniform(0, 5, len(cloud))))
    data.update(po_accum=stats2.accum.copy(), po_count=stats2.count.copy())
    cloud.opacity_logits = f32(cloud.opacity_logits)
    data["po_in_opacity"] = cloud.opacity_logits.copy()
    n_pruned = G.prune_only(cloud, stats2, cfg)
    data.update(po_pruned=n_pruned, po_out_accum=stats2.accum, po_out_count=stats2.count,
                po_out_positions=cloud.positions)
    cloud.opacity_logits = f32(cloud.opacity_logits)
    data["ro_in"] = cloud.opacity_logits.copy()
    G.reset_opacity(cloud, 0.01)
    data["ro_out"] = cloud.opacity_logits
    np.savez_compressed(os.path.join(OUT, "density.npz"), **data)
    print("density", rep)


def checkpoint_case(ref, seed=41):
    """An FS4C container written by the reference's own entry writer
    (training.py:599-628, the code save_checkpoint runs), plus its entries."""
    import io
    import struct
    T = ref["training"]
    rng = np.random.default_rng(seed)
    entries = {
        "meta.config": b"[train]\nseed = 3\n",
        "meta.iteration": 7,
        "meta.extent": 1.25,
        "meta.aabb": rng.normal(size=(2, 3)),
        "stats.accum": rng.uniform(size=11),
        "cloud.positions": rng.normal(size=(11, 3)),
        "cloud.opacity_logits": rng.normal(size=11),
        "grid.l0.p2": rng.normal(size=(4, 3, 2)),
        "net.trunk.0.weight": rng.normal(size=(5, 4)),
        "adam.positions.step": 3,
        "labels": np.arange(6, dtype=np.int64).reshape(2, 3),
    }
    buf = io.BytesIO()
    buf.write(T.CHECKPOINT_MAGIC)
    buf.write(struct.pack("<IQ", T.CHECKPOINT_VERSION, len(entries)))
    for name in sorted(entries):
        T._write_entry(buf, name, entries[name])
    with open(os.path.join(OUT, "checkpoint.fs4c"), "wb") as fh:
        fh.write(buf.getvalue())
    back = T.load_entries(os.path.join(OUT, "checkpoint.fs4c"))
    assert sorted(back) == sorted(entries)
    print("checkpoint", len(buf.getvalue()), "bytes")


def hexplane_edge_case(ref, name, t, seed=47):
    """HexPlane edge semantics (hexplane.py:84-110, 145-187; SURVEY Appendix A
    #11/#13): Gaussians outside the aabb along every axis (clamped coords, no
    dpos), Gaussians exactly on the lower and upper faces (raw = 0 / 1: the
    c = 1 cell is i0 = R-2, fa = 1), and t at the ends of [0, 1] (and beyond,
    clipped).  Stores the query, query_backward and the full deform /
    deform_backward through the reference."""
    H, D, G = ref["hexplane"], ref["deformation"], ref["gaussians"]
    rng = np.random.default_rng(seed)
    k, nf = 48, 8
    arrs = cloud_arrays(rng, k, nf, (0.15, 0.3), (2.2, 3.8))
    aabb = np.array([[-1.0, -1.0, 2.0], [1.0, 1.0, 4.0]])  # fp32-exact faces
    pos = arrs["positions"].copy()
    for i in range(12):                       # outside along each axis, both sides
        ax, side = i % 3, (i // 3) % 2
        pos[i, ax] = aabb[side, ax] + (0.25 + 0.1 * i) * (1 if side else -1)
    for i in range(12, 18):                   # exactly on a face
        ax, side = i % 3, (i // 3) % 2
        pos[i, ax] = aabb[side, ax]
    pos[18] = aabb[0]                         # both corners of the box
    pos[19] = aabb[1]
    pos[20] = aabb[1] + 0.5                   # outside on every axis
    arrs["positions"] = f32(pos)
    # 32 channels per plane and a width-64 depth-1 net: the shapes of the
    # tensor-core deformation path (the configs[1] kernels)
    field = H.HexPlaneField(H.HexPlaneConfig(levels=(1, 2), base_resolution=(6, 5, 7, 4), out_dim=64), aabb, rng)
    for li, level in enumerate(field.planes):
        for pi in range(len(level)):
            field.planes[li][pi] = f32(0.8 + rng.normal(size=level[pi].shape) * 0.3)
    net = D.DeformationNet(field.latent_dim, D.DeformationConfig(width=64, depth=1, feature_dim=nf), rng)
    for prefix, stack in net.stacks():
        for layer in stack:
            layer.weight = f32(rng.normal(size=layer.weight.shape) * 0.15)
            layer.bias = f32(rng.normal(size=layer.bias.shape) * 0.2)
    cloud = G.GaussianCloud(**{k_: v.copy() for k_, v in arrs.items()})
    lat, qcache = H.query_with_cache(field, cloud.positions, t)
    d_lat = f32(rng.normal(size=lat.shape))
    qpg, qdpos = H.query_backward(field, qcache, d_lat)
    coords, inside = field.normalized_coords(cloud.positions, t)
    snap, cache = D.deform_with_cache(cloud, field, net, t)
    ups = {n_: f32(rng.normal(size=np.shape(getattr(cloud, n_))))
           for n_ in ("positions", "rotations", "log_scales", "opacity_logits", "features")}

    class Gr:
        pass

    gr = Gr()
    for n_, v in ups.items():
        setattr(gr, n_, v)
    cg, ng, pg = D.deform_backward(cloud, field, net, cache, gr)
    data = {f"cloud_{k_}": v for k_, v in arrs.items()}
    data.update(aabb=aabb, t=t, width=64, depth=1, levels=np.asarray((1, 2)), base=np.asarray((6, 5, 7, 4)),
                out_dim=64, feature_dim=nf, latent=lat, d_latent=d_lat, query_dpos=qdpos, coords=coords,
                inside=inside)
    for li, level in enumerate(field.planes):
        for pi, pl in enumerate(level):
            data[f"plane_{li}_{pi}"] = pl
            data[f"qgplane_{li}_{pi}"] = qpg[li][pi]
            data[f"gplane_{li}_{pi}"] = pg[li][pi]
    for prefix, stack in net.stacks():
        for i, layer in enumerate(stack):
            data[f"w:{prefix}.{i}"] = layer.weight
            data[f"b:{prefix}.{i}"] = layer.bias
    for k_, v in ng.items():
        data[f"g:{k_}"] = v
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        data[f"snap_{f}"] = getattr(snap, f)
        data[f"up_{f}"] = ups[f]
    data["cg_positions"] = cg["positions"]
    np.savez_compressed(os.path.join(OUT, f"hexplane_{name}.npz"), **data)
    print("hexplane", name, "outside", int((~inside).any(axis=1).sum()))


def feature_map_case(ref, seed=43):
    """An FE4D teacher-feature file written by the reference's own
    save_feature_map (semantic.py:49-55)."""
    S = ref["semantic"]
    rng = np.random.default_rng(seed)
    fmap = S.FeatureMap(rng.normal(size=(3, 5, 7)).astype(np.float32))
    S.save_feature_map(os.path.join(OUT, "feature_map.feat"), fmap)
    print("feature map", fmap.data.shape)


def hexplane_edges(ref):
    hexplane_edge_case(ref, "t0", 0.0)
    hexplane_edge_case(ref, "t1", 1.0)
    hexplane_edge_case(ref, "tclip", 1.3)


def main():
    ref = load_reference()
    if len(sys.argv) > 1 and sys.argv[1] == "feature_map":
        feature_map_case(ref)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "hexplane_edges":
        hexplane_edges(ref)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "checkpoint":
        checkpoint_case(ref)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "train_ops":
        train_ops_case(ref)
        return
    if len(sys.argv) > 1 and sys.argv[1] == "density":
        density_case(ref)
        return
    train_ops_case(ref)
    density_case(ref)
    checkpoint_case(ref)
    feature_map_case(ref)
    hexplane_edges(ref)
    # the reference's own tiled-vs-naive scenes (test_rasterizer.py:168-183 sizes)
    render_case(ref, "s0", 0, 50, 32, 32, 4, 1.1 * 32, (0.1, 0.2, 0.3))
    render_case(ref, "s1", 1, 200, 64, 64, 16, 1.1 * 64, (0.1, 0.2, 0.3))
    render_case(ref, "s2", 2, 120, 48, 48, 4, 1.1 * 48, (0.1, 0.2, 0.3))
    render_case(ref, "s3", 3, 30, 33, 33, 16, 1.1 * 33, (0.1, 0.2, 0.3))
    # non-square, ragged tiles, rigid non-identity view (SURVEY §4 coverage gap)
    render_case(ref, "rigid", 7, 300, 40, 72, 8, 60.0, (0.0, 0.0, 0.0), rigid_T=True)
    # configs[0]-shaped, reduced K (fits in a small fixture): 160x128, fx=150, D=8
    render_case(ref, "cfg0", 11, 1500, 128, 160, 8, 150.0, (0.0, 0.0, 0.0),
                depth_range=(2.0, 4.0), op_range=(0.05, 0.95), with_backward=True,
                ls_range=(0.01, 0.05))
    # reference test_deformation.make_parts shapes
    deform_case(ref, "small", 5, 6, 5, 16, 3, (1, 2), (4, 4, 4, 3), 8)
    deform_case(ref, "wide", 6, 64, 16, 64, 1, (1, 2), (8, 8, 8, 5), 64)


if __name__ == "__main__":
    main()
