"""GPU parity of the deformation path (fs4d_deform_fwd / fs4d_deform_bwd through
deform / deform_with_cache / deform_backward) against golden vectors made by
the reference, and against the oracle at the BASELINE configs[1] shapes.

Tolerances (fp32 device vs fp64 reference): snapshot 1e-4 max-abs; gradients
1e-4 relative to the gradient scale (max(1, max|ref|))."""

import numpy as np
import pytest

from conftest import golden_cloud, has_gpu, load_golden, random_cloud_arrays
from oracle import fs4d_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def fs():
    import paper_2503_06161_b200 as m
    return m


def build_parts(g):
    m = fs()
    levels = tuple(int(x) for x in g["levels"])
    base = tuple(int(x) for x in g["base"])
    cfg = m.HexPlaneConfig(levels=levels, base_resolution=base, out_dim=int(g["out_dim"]))
    field = m.HexPlaneField(cfg, g["aabb"], np.random.default_rng(0))
    for l in range(len(levels)):
        for p in range(6):
            field.planes[l][p] = g[f"plane_{l}_{p}"]
    net = m.DeformationNet(field.latent_dim, m.DeformationConfig(width=int(g["width"]), depth=int(g["depth"]),
                                                                 feature_dim=int(g["feature_dim"])),
                           np.random.default_rng(0))
    for prefix, st in net.stacks():
        for i, layer in enumerate(st):
            layer.weight = g[f"w:{prefix}.{i}"]
            layer.bias = g[f"b:{prefix}.{i}"]
    c = golden_cloud(g)
    cloud = m.GaussianCloud(c.positions, c.rotations, c.log_scales, c.opacity_logits, c.colors_raw, c.features)
    return cloud, field, net


def close(a, b, what, rel=False):
    tol = TOL * (max(1.0, np.abs(b).max(initial=0.0)) if rel else 1.0)
    err = np.abs(np.asarray(a) - np.asarray(b)).max(initial=0.0)
    assert err < tol, (what, err, tol)


@pytest.mark.parametrize("case", ["small", "wide"])
def test_deform_matches_reference_golden(case):
    g = load_golden("deform_" + case)
    cloud, field, net = build_parts(g)
    t = float(g["t"])
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        close(getattr(snap, f), g[f"snap_{f}"], f)
    assert snap.colors_raw is cloud.colors_raw

    class G:
        pass

    gr = G()
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        setattr(gr, f, g[f"up_{f}"])
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, gr)
    close(cg["positions"], g["cg_positions"], "cloud positions", rel=True)
    assert cg["rotations"] is gr.rotations
    for key in g:
        if key.startswith("g:"):
            close(ng[key[2:]], g[key], key, rel=True)
    for l, level in enumerate(pg):
        for p, arr in enumerate(level):
            close(arr, g[f"gplane_{l}_{p}"], f"plane {l}/{p}", rel=True)


def test_flags_grid_disabled_and_feature_update_disabled():
    g = load_golden("deform_small")
    cloud, field, net = build_parts(g)
    net.cfg.enable_grid = False
    snap = fs().deform(cloud, field, net, 0.5)
    d = snap.positions - cloud.positions
    assert np.allclose(d, d[0], atol=1e-6)
    net.cfg.enable_grid = True
    net.cfg.enable_feature_update = False
    snap = fs().deform(cloud, field, net, 0.5)
    assert snap.features is cloud.features


def config1_parts(k=20000, seed=0):
    """BASELINE configs[1] shapes: levels (1,2), base (64,64,64,25), 32 ch, planes U[0.1,0.5],
    MLP width 64 depth 1 Xavier everywhere, D=16."""
    m = fs()
    rng = np.random.default_rng(seed)
    a = random_cloud_arrays(rng, k, 16, depth_range=(3.0, 6.0), xy=1.0)
    cloud = m.GaussianCloud(**{kk: v for kk, v in a.items() if kk != "sh_rest"})
    field = m.HexPlaneField(m.HexPlaneConfig(levels=(1, 2), base_resolution=(64, 64, 64, 25), out_dim=64),
                            m.scene_aabb(cloud), rng, init="uniform")
    for level in field.planes:
        for i in range(6):
            level[i] = level[i].astype(np.float32).astype(np.float64)
    net = m.DeformationNet(64, m.DeformationConfig(width=64, depth=1, feature_dim=16), rng, init="xavier",
                           head_init="xavier")
    for _, st in net.stacks():
        for layer in st:
            layer.weight = layer.weight.astype(np.float32).astype(np.float64)
    return cloud, field, net


def oracle_net(net):
    return {p: [(l.weight, l.bias, l.activation == "relu") for l in st] for p, st in net.stacks()}


# ReLU gates whose fp64 pre-activation lies within this relative band of 0 are
# ambiguous (the tensor-core path rounds operands to bf16x3, ~2^-17 relative);
# their Gaussians get zero upstream gradient so both sides agree on every
# surviving gate.
TAU_GATE = 1e-5


def gated_upstream(cloud, net, ocache, seed=1):
    rng = np.random.default_rng(seed)
    ups = {f: rng.normal(size=np.shape(getattr(cloud, f))).astype(np.float32).astype(np.float64)
           for f in ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    amb = O.relu_gate_margins(oracle_net(net), ocache) < TAU_GATE
    for f in ups:
        ups[f][amb] = 0.0
    return ups, int(amb.sum())


def test_config1_shapes_forward_and_backward_vs_oracle():
    cloud, field, net = config1_parts()
    t = 0.37
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    osnap, ocache = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        close(getattr(snap, f), osnap[f], f)
    ups, n_amb = gated_upstream(cloud, net, ocache)
    assert n_amb < 0.03 * len(cloud), n_amb
    gr = type("G", (), ups)()
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, gr)
    ocg, ong, opg = O.deform_backward(cloud, field.planes, field.aabb, oracle_net(net), ocache, ups)
    close(cg["positions"], ocg["positions"], "positions", rel=True)
    for k in ong:
        close(ng[k], ong[k], k, rel=True)
    for l in range(2):
        for p in range(6):
            close(pg[l][p], opg[l][p], f"plane {l}/{p}", rel=True)


def test_tc_backward_matches_recompute_path_at_full_size():
    """configs[1] size (200k Gaussians): the cached tensor-core backward and the
    recompute backward (no cache) agree on every gradient (ambiguous gates
    excluded as above)."""
    cloud, field, net = config1_parts(k=200_000, seed=3)
    t = 0.81
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    assert cache["device"] is not None and cache["device"].nbytes > 0
    _, ocache = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    ups, n_amb = gated_upstream(cloud, net, ocache, seed=4)
    assert n_amb < 0.03 * len(cloud), n_amb
    gr = type("G", (), ups)()
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, gr)
    plain = dict(cache)
    plain["device"] = None
    cg2, ng2, pg2 = fs().deform_backward(cloud, field, net, plain, gr)
    close(cg["positions"], cg2["positions"], "positions", rel=True)
    for k in ng:
        close(ng[k], ng2[k], k, rel=True)
    for l in range(2):
        for p in range(6):
            close(pg[l][p], pg2[l][p], f"plane {l}/{p}", rel=True)


@pytest.mark.parametrize("k", [0, 1, 127, 129])
def test_tc_backward_ragged_tiles(k):
    """Tile edges of the tensor-core backward: empty cloud, single Gaussian,
    one short tile, one full tile plus one row."""
    cloud, field, net = config1_parts(k=max(k, 1), seed=5)
    if k == 0:
        m = fs()
        cloud = m.GaussianCloud(*(np.zeros((0,) + np.shape(getattr(cloud, f))[1:]) for f in
                                  ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw",
                                   "features")))
    t = 0.5
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    _, ocache = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    ups = {f: np.random.default_rng(6).normal(size=np.shape(getattr(cloud, f))) for f in
           ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    if k:
        amb = O.relu_gate_margins(oracle_net(net), ocache) < TAU_GATE
        for f in ups:
            ups[f][amb] = 0.0
    gr = type("G", (), ups)()
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, gr)
    ocg, ong, opg = O.deform_backward(cloud, field.planes, field.aabb, oracle_net(net), ocache, ups)
    close(cg["positions"], ocg["positions"], "positions", rel=True)
    for key in ong:
        close(ng[key], ong[key], key, rel=True)
    for l in range(2):
        for p in range(6):
            close(pg[l][p], opg[l][p], f"plane {l}/{p}", rel=True)


def test_cache_from_another_time_is_a_contract_violation():
    from paper_2503_06161_b200.errors import ContractViolation
    cloud, field, net = config1_parts(k=300, seed=7)
    _, cache = fs().deform_with_cache(cloud, field, net, 0.25)
    _, other = fs().deform_with_cache(cloud, field, net, 0.75)
    bad = dict(cache)
    bad["device"] = other["device"]
    ups = {f: np.ones(np.shape(getattr(cloud, f))) for f in
           ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    with pytest.raises(ContractViolation):
        fs().deform_backward(cloud, field, net, bad, type("G", (), ups)())


def test_locality_order_is_a_permutation_and_changes_nothing():
    """fs4d_locality_order (Morton order of the canonical positions) is a
    permutation of [0, K); deforming with it (Fs4dHexPlane.order) gives
    bit-identical snapshots, since every Gaussian's latent is computed
    independently."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv

    rng = np.random.default_rng(17)
    k = 20_000
    a = random_cloud_arrays(rng, k, 16, depth_range=(2.0, 4.0), xy=1.0)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(16, 16, 16, 5), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=16), rng, init="xavier",
                            head_init="xavier")
    c, f, n = dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net)
    order = dv.locality_order(c.positions, f.aabb)
    o = order.cpu().numpy()
    np.testing.assert_array_equal(np.sort(o), np.arange(k))
    # Morton order: consecutive Gaussians are spatially close on average
    p = a["positions"]
    assert np.linalg.norm(np.diff(p[o], axis=0), axis=1).mean() < 0.2 * np.linalg.norm(np.diff(p, axis=0), axis=1).mean()
    e = dv.DeformEngine()
    s0 = e.forward(c, f, n, 0.43)
    s1 = e.forward(c, f.with_order(order), n, 0.43)
    torch.cuda.synchronize()
    for name in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        assert torch.equal(getattr(s0, name), getattr(s1, name)), name


@pytest.mark.parametrize("case", ["t0", "t1", "tclip"])
def test_hexplane_edges_match_reference_golden(case):
    """Outside-aabb Gaussians (clamped coordinates, no dpos), Gaussians on the
    aabb faces (c = 1 -> i0 = R-2, fa = 1) and t = 0 / 1 / 1.3 (clipped),
    through the tensor-core deformation path (32 channels, width 64): forward
    and backward against reference goldens (make_golden.hexplane_edge_case;
    hexplane.py:84-110, 186)."""
    g = load_golden("hexplane_" + case)
    cloud, field, net = build_parts(g)
    t = float(g["t"])
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    assert cache["device"] is not None and cache["device"].nbytes > 0  # the cached tensor-core backward
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        close(getattr(snap, f), g[f"snap_{f}"], f)
    gr = type("G", (), {f: g[f"up_{f}"] for f in ("positions", "rotations", "log_scales", "opacity_logits",
                                                 "features")})()
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, gr)
    close(cg["positions"], g["cg_positions"], "cloud positions", rel=True)
    outside = ~g["inside"]
    # rows with every axis clamped get exactly the upstream position gradient
    allout = outside.all(axis=1)
    assert allout.any()
    np.testing.assert_array_equal(cg["positions"][allout], np.asarray(g["up_positions"], np.float32)[allout])
    for key in g:
        if key.startswith("g:"):
            close(ng[key[2:]], g[key], key, rel=True)
    for l, level in enumerate(pg):
        for p, arr in enumerate(level):
            close(arr, g[f"gplane_{l}_{p}"], f"plane {l}/{p}", rel=True)


@pytest.mark.parametrize("t", [0.0, 1.0])
def test_config1_shapes_outside_aabb_and_time_ends_vs_oracle(t):
    """configs[1] plane / MLP shapes with a shrunken aabb (about a third of the
    Gaussians clamped on some axis) at t = 0 and t = 1: forward and backward
    against the oracle, ambiguous ReLU gates excluded as above."""
    cloud, field, net = config1_parts(k=20000, seed=11)
    lo, hi = field.aabb
    field.aabb = np.stack([lo + 0.12 * (hi - lo), hi - 0.12 * (hi - lo)])
    _, inside = O.field_coords(field.aabb, cloud.positions, t)
    assert 0.2 < (~inside).any(axis=1).mean() < 0.8
    snap, cache = fs().deform_with_cache(cloud, field, net, t)
    osnap, ocache = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        close(getattr(snap, f), osnap[f], f)
    ups, n_amb = gated_upstream(cloud, net, ocache, seed=12)
    assert n_amb < 0.03 * len(cloud), n_amb
    cg, ng, pg = fs().deform_backward(cloud, field, net, cache, type("G", (), ups)())
    ocg, ong, opg = O.deform_backward(cloud, field.planes, field.aabb, oracle_net(net), ocache, ups)
    close(cg["positions"], ocg["positions"], "positions", rel=True)
    for k in ong:
        close(ng[k], ong[k], k, rel=True)
    for l in range(2):
        for p in range(6):
            close(pg[l][p], opg[l][p], f"plane {l}/{p}", rel=True)


@pytest.mark.parametrize("k", [1, 127, 129, 383, 20000])
def test_two_slot_forward_ragged_sizes_vs_oracle(k):
    """The forward without cache (k_mlp_tc_2s: two tile pipelines per CTA, the
    latent as TMA-loaded bf16 rows, rows past K zero-filled by the TMA unit):
    one row, a short tile, a tile plus one row, an odd number of tiles (the
    second slot of the last CTA idle) and a configs[1]-shaped batch, against
    the oracle; and bitwise equal to deform_with_cache's forward (the cached
    path writes the same snapshot)."""
    cloud, field, net = config1_parts(k=k, seed=7)
    t = 0.61
    snap = fs().deform(cloud, field, net, t)
    snap_c, _ = fs().deform_with_cache(cloud, field, net, t)
    osnap, _ = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        close(getattr(snap, f), osnap[f], f)
        assert np.array_equal(np.asarray(getattr(snap, f)), np.asarray(getattr(snap_c, f))), f
