"""Parity at the BASELINE headline configurations against
the float64 oracle, at full size.

* configs[1] (the bench workload itself, bench.make_scene: 200k Gaussians,
  640x512, fx=fy=560, SH3, D=16, HexPlane (1,2)x(64,64,64,25)x32, Xavier MLP
  width 64) at t = 0, 0.37 and 1: device deform vs oracle deform, then the
  device render of the device snapshot vs the oracle render of the SAME fp32
  snapshot (stage injection, §8(c) rule 4).  Visible set, radius, depth order
  and every tile list are compared full-frame; images and per-pixel
  contributor counts on the composited tile rows (all rows at t = 0.37, every
  other row at t = 0 / 1 to bound the oracle's time).
* configs[3] (500k Gaussians, 1280x1024, fx=fy=1100, SH3, D=32): the same
  for one frame, every fourth tile row composited.
* configs[4] (training step): TrainStep over 2 (view, t) pairs of the
  configs[1] scene with rigid views, L1 RGB + L1 feature loss against random
  targets, against the oracle chain (deform -> render -> L1 -> render_backward
  -> deform_backward) run on each pair's device snapshot; every gradient of
  the flat all-reduce buffer is compared.

Contract: discrete decisions match exactly wherever the deciding quantity is
not within a relative margin TAU (fp32 blend decisions) / TAU64 (fp64
projection decisions) of its flip point; ambiguous Gaussians are removed from
both sides' lists before comparing, ambiguous pixels (dilated by the
footprint of ambiguous Gaussians) are excluded from the image comparison,
and Gaussians whose footprint covers an ambiguous pixel (or whose ReLU gates
are ambiguous) from the per-Gaussian gradient comparison.  Every exclusion
is counted and printed.  Images: 1e-4 max-abs; gradients: 1e-4 x max|g| per
tensor (the loss normalisation makes these gradients ~1e-6, so an absolute
1e-4 would be vacuous).
"""

import numpy as np
import pytest

from conftest import has_gpu, pinhole, rigid_T
from oracle import fs4d_oracle as O

pytestmark = pytest.mark.gpu

TAU = 1e-5
# The stop rule compares the fp32 transmittance, a product over every earlier
# contributor, with 1e-4: with ~50-130 contributors per pixel its relative
# error reaches ~1e-5 (sum of alpha_i/(1-alpha_i) ~ ln(1e4) times the ~1e-6
# relative alpha error), so stop decisions get a 10x wider band than the
# per-Gaussian alpha decisions.
TAU_STOP = 1e-4
TAU64 = 1e-9
TAU_GATE = 1e-5
ATOL_IMG = 1e-4
RTOL_GRAD = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def fs():
    import paper_2503_06161_b200 as m
    return m


class _C:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def oracle_net(net):
    return {p: [(l.weight, l.bias, l.activation == "relu") for l in st] for p, st in net.stacks()}


@pytest.fixture(scope="module")
def config1():
    import bench
    return bench.make_scene(0)


def config3_scene(seed=3):
    """configs[3]: SCARED-shaped, same distributions as bench.make_scene."""
    m = fs()
    rng = np.random.default_rng(seed)
    k, d = 500_000, 32
    f32 = lambda x: np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = rng.normal(0.0, 0.2, size=(k, 16, 3))
    cloud = m.GaussianCloud(
        positions=f32(np.column_stack([rng.uniform(-1, 1, k), rng.uniform(-1, 1, k), rng.uniform(3, 6, k)])),
        rotations=f32(q), log_scales=f32(rng.normal(-4.0, 0.5, size=(k, 3))),
        opacity_logits=f32(rng.normal(0.0, 1.0, size=k)), colors_raw=f32(sh[:, 0, :]),
        features=f32(rng.normal(size=(k, d))), sh_rest=f32(sh[:, 1:, :]))
    field = m.HexPlaneField(m.HexPlaneConfig(levels=(1, 2), base_resolution=(64, 64, 64, 25), out_dim=64),
                            m.scene_aabb(cloud), rng, init="uniform")
    for level in field.planes:
        for i in range(6):
            level[i] = f32(level[i])
    net = m.DeformationNet(64, m.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                           head_init="xavier")
    for _, st in net.stacks():
        for layer in st:
            layer.weight = f32(layer.weight)
    return cloud, field, net, pinhole(1024, 1280, 1100.0)


def make_frame(K, T, h, w, time=0.0):
    return fs().CameraFrame(K=K, T=T, time=time, image=np.zeros((h, w, 3)), depth=np.zeros((h, w)),
                            mask=np.ones((h, w), dtype=bool))


def snapshot_obj(snap):
    return _C(**{f: np.asarray(getattr(snap, f)) for f in ("positions", "rotations", "log_scales",
                                                          "opacity_logits", "colors_raw", "features")},
              sh_rest=getattr(snap, "sh_rest", None))


def ambiguity(oout, cfg, h, w, split=False):
    """(ambiguous pixel mask, ambiguous source indices): pixels that met an
    fp32 blend decision within TAU (stop rule: TAU_STOP), dilated by the
    footprint of every Gaussian with an fp64 projection decision within
    TAU64.  split=True returns (alpha/projection-ambiguous pixels,
    stop-only-ambiguous pixels, sources)."""
    proj = oout["proj"]
    m_alpha, m_stop = O.pixel_decision_margins(oout, cfg, split=True)
    amb = m_alpha < TAU
    amb_stop = m_stop < TAU_STOP
    if not split:
        amb = amb | amb_stop
    pm = O.projection_margins(proj, h, w, cfg.tile, cfg)
    amb_g = pm < TAU64
    for g in np.flatnonzero(amb_g):
        u, v, r = proj["mean2d"][g, 0], proj["mean2d"][g, 1], proj["radius"][g]
        x0, x1 = int(max(0, np.floor(u - r - 1))), int(min(w - 1, np.ceil(u + r + 1)))
        y0, y1 = int(max(0, np.floor(v - r - 1))), int(min(h - 1, np.ceil(v + r + 1)))
        amb[y0:y1 + 1, x0:x1 + 1] = True
    src = set(proj["source_index"][amb_g].tolist())
    return (amb, amb_stop & ~amb, src) if split else (amb, src)


def compare_frame(snap, K, T, h, w, tile_rows, label):
    """Device render vs oracle render of the same fp32 snapshot."""
    cfg, ocfg = fs().RasterConfig(), O.RasterParams()
    out = fs().render(snap, make_frame(K, T, h, w), cfg)
    osnap = snapshot_obj(snap)
    oproj = O.project(osnap, K, T, h, w, ocfg)
    olists = O.bin_tiles(oproj, h, w, 16)
    oout = O.render(osnap, K, T, h, w, ocfg, tile_rows=tile_rows, prepared=(oproj, olists), margins=True)
    amb, amb_src = ambiguity(oout, ocfg, h, w)

    # visible set and radius (fp64 on device: exact)
    gproj = out.record.proj
    assert np.array_equal(np.sort(gproj.source_index), np.sort(oproj["source_index"])), label
    g_of = np.empty(len(snap.positions), dtype=np.int64)
    g_of[gproj.source_index] = np.arange(len(gproj.source_index))
    keep_g = ~np.isin(oproj["source_index"], list(amb_src))
    rad_dev = gproj.radius[g_of[oproj["source_index"]]]
    assert np.array_equal(rad_dev[keep_g], oproj["radius"][keep_g]), label
    # depth order of the non-ambiguous Gaussians
    drop = np.isin(gproj.source_index, list(amb_src))
    assert np.array_equal(gproj.source_index[~drop], oproj["source_index"][keep_g]), label
    # every tile list, as source indices in depth order
    glists = out.record.tile_lists()
    n_pairs = n_cmp = 0
    for ty, row in enumerate(olists):
        for tx, cell in enumerate(row):
            osrc = oproj["source_index"][cell]
            gsrc = gproj.source_index[glists[ty][tx]]
            osrc = osrc[~np.isin(osrc, list(amb_src))]
            gsrc = gsrc[~np.isin(gsrc, list(amb_src))]
            assert np.array_equal(gsrc, osrc), (label, ty, tx)
            n_pairs += cell.size
            n_cmp += 1
    # images + contributor counts on the composited rows
    rows = np.zeros(h, dtype=bool)
    for ty in tile_rows:
        rows[ty * 16:min(h, ty * 16 + 16)] = True
    ok = ~amb & rows[:, None]
    m_alpha, m_stop = O.pixel_decision_margins(oout, O.RasterParams(), split=True)
    for key in ("color", "depth", "feature", "alpha"):
        diff = np.abs(getattr(out, key) - oout[key])
        if diff.ndim == 3:
            diff = diff.max(axis=2)
        bad = np.argwhere(ok & (diff >= ATOL_IMG))
        if bad.size:
            i, j = bad[0]
            raise AssertionError(f"{label} {key}: {len(bad)} pixels off, first ({i},{j}) diff {diff[i, j]:.3g} "
                                 f"n_contrib dev {out.n_contrib[i, j]} ref {oout['n_contrib'][i, j]} "
                                 f"alpha margin {m_alpha[i, j]:.3g} stop margin {m_stop[i, j]:.3g}")
    nbad = int((ok & (out.n_contrib != oout["n_contrib"])).sum())
    assert nbad == 0, (label, "n_contrib differs on", nbad, "non-ambiguous pixels")
    print(f"[{label}] visible {len(gproj)}  pairs {n_pairs} in {n_cmp} tiles (all compared)  "
          f"ambiguous Gaussians {len(amb_src)}  composited pixels {int(rows.sum()) * w}  "
          f"ambiguous pixels excluded {int((amb & rows[:, None]).sum())}")
    return out, oout


@pytest.mark.parametrize("t", [0.0, 0.37, 1.0])
def test_config1_full_frame_deform_and_render_vs_oracle(config1, t):
    cloud, field, net, K = config1
    h, w = 512, 640
    snap = fs().deform(cloud, field, net, t)
    osnap, ocache = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        err = np.abs(np.asarray(getattr(snap, f)) - osnap[f]).max()
        assert err < 1e-4, (f, err)
    assert snap.sh_rest is cloud.sh_rest and snap.colors_raw is cloud.colors_raw
    nty = -(-h // 16)
    rows = range(nty) if t == 0.37 else range(0, nty, 2)
    compare_frame(snap, K, np.eye(4), h, w, rows, f"configs[1] t={t}")


def test_config3_frame_vs_oracle():
    cloud, field, net, K = config3_scene()
    h, w = 1024, 1280
    t = 0.58
    snap = fs().deform(cloud, field, net, t)
    osnap, _ = O.deform(cloud, field.planes, field.aabb, oracle_net(net), t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        err = np.abs(np.asarray(getattr(snap, f)) - osnap[f]).max()
        assert err < 1e-4, (f, err)
    compare_frame(snap, K, np.eye(4), h, w, range(0, -(-h // 16), 4), "configs[3]")


def test_config4_training_gradients_vs_oracle_chain(config1):
    """configs[4] at full size: 2 (view, t) pairs through TrainStep, every
    gradient of the flat all-reduce buffer against the oracle chain, in two
    stages so that each comparison is exact up to fp32 arithmetic:

    * render stage: each pair's device snapshot gradients (the lane's
      render-backward output) against the oracle's render_backward of the same
      fp32 snapshot with the same L1 upstream -- per Gaussian, excluding the
      Gaussians an ambiguous decision can touch;
    * deformation stage: the oracle's deform_backward fed the DEVICE's
      snapshot gradients against the flat buffer's cloud / plane / MLP
      gradients (summed over the pairs) -- every entry, no exclusions.

    The end-to-end aggregate error (oracle chain vs device) is reported too."""
    import torch
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.train import TrainStep

    cloud, field, net, K = config1
    h, w, d = 512, 640, 16
    k = len(cloud)
    rng = np.random.default_rng(404)
    views = [(0.23, rigid_T(rng)), (0.81, rigid_T(rng))]
    targets = [(rng.uniform(size=(h, w, 3)).astype(np.float32), rng.normal(size=(h, w, d)).astype(np.float32))
               for _ in views]
    step = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                     h, w, fs().RasterConfig(), lanes=2)
    batch = [(t, K, T, torch.as_tensor(tr, device="cuda"), torch.as_tensor(tf, device="cuda"))
             for (t, T), (tr, tf) in zip(views, targets)]
    loss = float(step.run(batch, check=True).item())
    torch.cuda.synchronize()
    host = lambda x: x.detach().cpu().numpy().astype(np.float64)  # noqa: E731
    snaps = [{f: host(getattr(ln.snap, f)) for f in ("positions", "rotations", "log_scales", "opacity_logits",
                                                       "features")} for ln in step._lanes]
    sgrads = [{f: host(getattr(ln.snap_grads, f)) for f in ("positions", "rotations", "log_scales", "opacity_logits",
                                                            "colors_raw", "sh_rest", "features")}
              for ln in step._lanes]

    onet = oracle_net(net)
    cfg = O.RasterParams()
    wpair = 1.0 / len(views)
    inj, chain, loss_ref = {}, {}, 0.0
    bad = np.zeros(k, dtype=bool)
    worst_render = worst_deform = 0.0

    def add(acc, key, v):
        acc[key] = acc.get(key, 0.0) + v

    for (t, T), (tr, tf), sd, sg in zip(views, targets, snaps, sgrads):
        osnap, ocache = O.deform(cloud, field.planes, field.aabb, onet, t)
        for f in sd:
            assert np.abs(sd[f] - osnap[f]).max() < 1e-4, f
        so = _C(**sd, colors_raw=cloud.colors_raw, sh_rest=cloud.sh_rest)
        out = O.render(so, K, T, h, w, cfg, margins=True)
        dcol, dfe = out["color"] - tr, out["feature"] - tf
        loss_ref += wpair * (np.abs(dcol).mean() + np.abs(dfe).sum() / (h * w))
        g = O.render_backward(so, K, T, h, w, cfg, out, wpair * np.sign(dcol) / (3 * h * w), None,
                              wpair * np.sign(dfe) / (h * w), None)
        # exclusions: Gaussians reached by the traversal of a pixel with an
        # ambiguous blend / projection decision or an ambiguous L1 sign, the
        # ambiguous projections themselves
        amb, amb_stop, amb_src = ambiguity(out, cfg, h, w, split=True)
        amb |= (np.abs(dcol) < 1e-5).any(axis=2) | (np.abs(dfe) < 1e-5).any(axis=2)
        pb = np.zeros(k, dtype=bool)
        pb[out["proj"]["source_index"][O.reached_rows(out, cfg, amb, amb_stop)]] = True
        pb[list(amb_src)] = True
        bad |= pb
        for f in sg:  # render stage, per Gaussian
            ref = np.asarray(g[f])
            tol = RTOL_GRAD * max(np.abs(ref).max(), 1e-30)
            err = np.abs(sg[f] - ref)[~pb].max()
            worst_render = max(worst_render, err / tol)
            assert err < tol, ("render stage", f, err, tol)
        # deformation stage on the device's snapshot gradients (stage
        # injection): the same gradients through fs.deform_backward and the
        # oracle, with the rows of Gaussians whose ReLU gates sit within
        # TAU_GATE of zero zeroed on both sides (their gate may resolve
        # either way in the tensor-core bf16x3 arithmetic)
        gate_amb = O.relu_gate_margins(onet, ocache) < TAU_GATE
        sgz = {f: np.where(gate_amb.reshape((-1,) + (1,) * (v.ndim - 1)), 0.0, v) for f, v in sg.items()}
        _, dcache = fs().deform_with_cache(cloud, field, net, t)
        dcg, dng, dpg = fs().deform_backward(cloud, field, net, dcache, _C(**sgz))
        ocg, ong, opg = O.deform_backward(cloud, field.planes, field.aabb, onet, ocache, sgz)
        for key, got, ref in ([("positions", dcg["positions"], ocg["positions"])] +
                              [(n, dng[n], ong[n]) for n in ong] +
                              [(f"grid.l{l}.p{p}", dpg[l][p], opg[l][p]) for l in range(2) for p in range(6)]):
            tol = max(RTOL_GRAD * np.abs(ref).max(), 1e-30)
            err = np.abs(got - ref).max()
            worst_deform = max(worst_deform, err / tol)
            assert err < tol, ("deformation stage", key, err, tol)
        # the training step's flat buffer is the sum over pairs of exactly
        # these device stages (unzeroed)
        ucg, ung, upg = fs().deform_backward(cloud, field, net, dcache, _C(**sg))
        add(inj, "positions", ucg["positions"])
        for f in ("rotations", "log_scales", "opacity_logits", "colors_raw", "sh_rest", "features"):
            add(inj, f, sg[f])
        for key, v in ung.items():
            add(inj, key, v)
        for l, level in enumerate(upg):
            for p, arr in enumerate(level):
                add(inj, f"grid.l{l}.p{p}", arr)
        # the full oracle chain, for the end-to-end report
        cg2, ng2, pg2 = O.deform_backward(cloud, field.planes, field.aabb, onet, ocache, g)
        add(chain, "positions", cg2["positions"])
        for key, v in ng2.items():
            add(chain, key, v)
        for l, level in enumerate(pg2):
            for p, arr in enumerate(level):
                add(chain, f"grid.l{l}.p{p}", arr)

    assert abs(loss - loss_ref) < 1e-5 * max(1.0, abs(loss_ref)), (loss, loss_ref)
    print(f"[configs[4]] render stage: {int(bad.sum())} of {k} Gaussians excluded, worst err/tol {worst_render:.2f}")
    worst = 0.0
    for key, ref in inj.items():  # the flat buffer == the per-pair device stages summed
        got = step.grads[key].cpu().numpy().astype(np.float64).reshape(np.shape(ref))
        tol = max(1e-5 * np.abs(ref).max(), 1e-30)
        err = np.abs(got - ref).max()
        worst = max(worst, err / tol)
        assert err < tol, ("training-step assembly", key, err, tol)
    # end to end (the oracle chain on its own snapshot gradients): differs
    # from the device by the ambiguous decisions excluded above, reported
    rel = {key: np.linalg.norm(step.grads[key].cpu().numpy().astype(np.float64).reshape(np.shape(v)) - v)
           / max(np.linalg.norm(v), 1e-30) for key, v in chain.items()}
    wkey = max(rel, key=rel.get)
    print(f"[configs[4]] deformation stage worst err/tol {worst_deform:.2f}; assembly worst err/tol {worst:.2f}; "
          f"end-to-end (oracle chain) aggregate rel. L2 error: median {np.median(list(rel.values())):.1e}, "
          f"worst {rel[wkey]:.1e} ({wkey})")
    assert rel[wkey] < 5e-2
