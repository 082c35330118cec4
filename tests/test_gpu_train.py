"""GPU parity of the configs[4]-style training step (paper_2503_06161_b200.train):
deform -> render -> fused L1 loss -> render_backward -> deform_backward,
accumulated over (view, t) pairs into the flat gradient buffer, against the
float64 oracle chained the same way.  Tolerance: 1e-3 x max|grad| per
tensor (relative; the loss normalisation makes gradients ~1e-5); Gaussians touching a pixel with an ambiguous fp32 blend decision
are excluded from the per-Gaussian comparison."""

import numpy as np
import pytest

from conftest import has_gpu, pinhole, random_cloud_arrays, rigid_T
from oracle import fs4d_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


class _C:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def test_train_step_matches_oracle_chain():
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.train import TrainStep

    rng = np.random.default_rng(42)
    k, h, w, d = 2500, 64, 96, 8
    a = random_cloud_arrays(rng, k, d, op_range=(0.05, 0.9), depth_range=(2.0, 4.0), xy=1.0,
                            ls_range=(np.exp(-4.0), np.exp(-2.8)), sh_degree=3)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(16, 16, 16, 5), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    for level in field.planes:
        for i in range(6):
            level[i] = (level[i] * 2.0).astype(np.float32).astype(np.float64)
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    for _, st in net.stacks():
        for layer in st:
            layer.weight = layer.weight.astype(np.float32).astype(np.float64)
    onet = {p: [(l.weight, l.bias, l.activation == "relu") for l in st] for p, st in net.stacks()}
    K = pinhole(h, w, 70.0)
    views = [(0.2, np.eye(4)), (0.7, rigid_T(rng))]
    cfg = O.RasterParams()
    pairs = []
    for t, T in views:
        snap, cache = O.deform(_C(**a), field.planes, field.aabb, onet, t)
        snap_obj = _C(**snap, sh_rest=a["sh_rest"])
        out = O.render(snap_obj, K, T, h, w, cfg)
        s_rgb = np.where(rng.random((h, w, 3)) < 0.5, -1.0, 1.0)
        s_f = np.where(rng.random((h, w, d)) < 0.5, -1.0, 1.0)
        tgt_rgb = (out["color"] - 0.25 * s_rgb).astype(np.float32)
        tgt_f = (out["feature"] - 0.5 * s_f).astype(np.float32)
        pairs.append((t, T, snap_obj, cache, out, tgt_rgb, tgt_f))

    # ---- device step ----
    dc = dv.DeviceCloud.from_cloud(cloud)
    step = TrainStep(dc, dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net), h, w, fs.RasterConfig())
    batch = [(t, K, T, torch.as_tensor(tr, device="cuda"), torch.as_tensor(tf, device="cuda"))
             for (t, T, _, _, _, tr, tf) in pairs]
    loss = float(step.run(batch, check=True).item())
    torch.cuda.synchronize()

    # ---- oracle chain ----
    wpair = 1.0 / len(pairs)
    acc = {}
    loss_ref = 0.0
    bad = np.zeros(k, dtype=bool)
    for (t, T, snap_obj, cache, out, tr, tf) in pairs:
        dcol = out["color"] - tr
        dfe = out["feature"] - tf
        loss_ref += wpair * (np.abs(dcol).mean() + np.abs(dfe).sum() / (h * w))
        gC = wpair * np.sign(dcol) / (3 * h * w)
        gF = wpair * np.sign(dfe) / (h * w)
        g = O.render_backward(snap_obj, K, T, h, w, cfg, out, gC, None, gF, None)
        cg, ng, pg = O.deform_backward(_C(**a), field.planes, field.aabb, onet, cache, g)
        contrib = {"positions": cg["positions"], "rotations": g["rotations"], "log_scales": g["log_scales"],
                   "opacity_logits": g["opacity_logits"], "colors_raw": g["colors_raw"],
                   "sh_rest": g["sh_rest"], "features": g["features"]}
        contrib.update(ng)
        for l, level in enumerate(pg):
            for p, arr in enumerate(level):
                contrib[f"grid.l{l}.p{p}"] = arr
        for key, v in contrib.items():
            acc[key] = acc.get(key, 0.0) + v
        amb = O.pixel_decision_margins(out, cfg) < 1e-5
        for (ty, tx), (rows, xs, ys) in out["tiles"].items():
            if amb[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1].any():
                bad[out["proj"]["source_index"][rows]] = True

    assert abs(loss - loss_ref) < 1e-5 * max(1.0, abs(loss_ref))
    keep = ~bad
    assert keep.mean() > 0.5
    for key, ref in acc.items():
        got = step.grads[key].cpu().numpy().astype(np.float64).reshape(np.shape(ref))
        if np.shape(ref)[0] == k and key in ("positions", "rotations", "log_scales", "opacity_logits",
                                               "colors_raw", "sh_rest", "features"):
            got, ref = got[keep], np.asarray(ref)[keep]
        # the 1/(3HW) loss normalisation makes these gradients small, so the
        # check is relative to each tensor's scale (stricter than 1e-4 absolute)
        tol = max(1e-3 * np.abs(ref).max(), 1e-12)
        assert np.abs(got - ref).max() < tol, (key, np.abs(got - ref).max(), tol)


def test_fine_stage_step_decoder_tv_adam_matches_oracle():
    """The reference's fine-stage iteration (training.py:489-535) on device:
    masked photometric + depth L1, pointwise-decoder feature loss against a
    half-resolution teacher, HexPlane TV, flat all-reduce buffer, then the
    multi-segment Adam step -- against the float64 oracle chained the same
    way (the Adam update is checked on the device's own gradients)."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.numerics import LrSchedule
    from paper_2503_06161_b200.optim import adam_eps, schedule_key
    from paper_2503_06161_b200.train import TrainStep

    rng = np.random.default_rng(7)
    k, h, w, d, ct = 2000, 64, 80, 8, 12
    ho, wo = 32, 40
    a = random_cloud_arrays(rng, k, d, op_range=(0.05, 0.9), depth_range=(2.0, 4.0), xy=1.0,
                            ls_range=(np.exp(-4.0), np.exp(-2.8)), sh_degree=1)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=32),
                             fs.scene_aabb(cloud), rng, init="uniform")
    for level in field.planes:
        for i in range(6):
            level[i] = (level[i] * 2.0).astype(np.float32).astype(np.float64)
    net = fs.DeformationNet(32, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    for _, st in net.stacks():
        for layer in st:
            layer.weight = layer.weight.astype(np.float32).astype(np.float64)
    onet = {p: [(l.weight, l.bias, l.activation == "relu") for l in st] for p, st in net.stacks()}
    dec_w = rng.uniform(-1, 1, size=(ct, d)).astype(np.float32).astype(np.float64)
    dec_b = (rng.normal(size=ct) * 0.1).astype(np.float32).astype(np.float64)
    K = pinhole(h, w, 60.0)
    lam_rgb, lam_d, lam_f, lam_tv = 1.0, 0.2, 0.7, 0.05
    cfg = O.RasterParams()
    pairs = []
    for t, T in ((0.3, np.eye(4)), (0.8, rigid_T(rng))):
        snap, cache = O.deform(_C(**a), field.planes, field.aabb, onet, t)
        snap_obj = _C(**snap, sh_rest=a["sh_rest"])
        out = O.render(snap_obj, K, T, h, w, cfg)
        assert np.abs(out["alpha"] - 0.5).min() > 1e-6  # no ambiguous depth-mask pixel
        sgn = lambda shape: np.where(rng.random(shape) < 0.5, -1.0, 1.0)  # noqa: E731
        tgt_rgb = (out["color"] - 0.25 * sgn((h, w, 3))).astype(np.float32)
        tgt_depth = (out["depth"] - 0.3 * sgn((h, w))).astype(np.float32)
        mask = rng.random((h, w)) > 0.2
        dec, _ = O.decoder_forward(dec_w, dec_b, out["feature"], (ho, wo))
        teacher = (dec - 0.5 * sgn((ho, wo, ct))).astype(np.float32)
        pairs.append((t, T, snap_obj, cache, out, tgt_rgb, tgt_depth, mask, teacher))

    # ---- device step ----
    f = dict(device="cuda")
    dec_dev = (torch.tensor(dec_w, dtype=torch.float32, **f), torch.tensor(dec_b, dtype=torch.float32, **f))
    step = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                     h, w, fs.RasterConfig(), loss_mode="decoder", lambda_rgb=lam_rgb, lambda_depth=lam_d,
                     lambda_feat=lam_f, lambda_tv=lam_tv, decoder=dec_dev)
    schedules = {"positions": LrSchedule(1.6e-4, 1.6e-6, 100), "rotations": LrSchedule.constant(1e-3),
                 "log_scales": LrSchedule.constant(5e-3), "opacity_logits": LrSchedule.constant(5e-2),
                 "colors_raw": LrSchedule.constant(2.5e-3), "features": LrSchedule.constant(2.5e-3),
                 "grid": LrSchedule(1.6e-3, 1.6e-5, 100), "net": LrSchedule(1.6e-4, 1.6e-6, 100, 0.01, 10),
                 "decoder": LrSchedule.constant(1e-3)}
    step.attach_optimizer(schedules)
    p0 = step.params.buffer.clone()
    batch = [(t, K, T, torch.as_tensor(tr, **f), torch.as_tensor(te, **f), torch.as_tensor(m, **f),
              torch.as_tensor(td, **f)) for (t, T, _, _, _, tr, td, m, te) in pairs]
    loss = float(step.run(batch, check=True).item())
    torch.cuda.synchronize()

    # ---- oracle chain ----
    wp = 1.0 / len(pairs)
    acc, loss_ref = {}, 0.0
    bad = np.zeros(k, dtype=bool)
    for (t, T, snap_obj, cache, out, tr, td, m, te) in pairs:
        rgb, dterm, gC, gD = O.photometric(out["color"], tr, m, out["depth"], td, out["alpha"], wp * lam_rgb,
                                           wp * lam_d)
        dec, resized = O.decoder_forward(dec_w, dec_b, out["feature"], (ho, wo))
        fl, d_dec = O.l1_mean_pixels(dec, te)
        gF, dW, dB = O.decoder_backward(dec_w, resized, (h, w), wp * lam_f * d_dec)
        loss_ref += wp * (lam_rgb * rgb + lam_d * dterm + lam_f * fl)
        g = O.render_backward(snap_obj, K, T, h, w, cfg, out, gC, gD, gF, None)
        cg, ng, pg = O.deform_backward(_C(**a), field.planes, field.aabb, onet, cache, g)
        contrib = {"positions": cg["positions"], "rotations": g["rotations"], "log_scales": g["log_scales"],
                   "opacity_logits": g["opacity_logits"], "colors_raw": g["colors_raw"],
                   "sh_rest": g["sh_rest"], "features": g["features"], "decoder.weight": dW, "decoder.bias": dB}
        contrib.update(ng)
        for l, level in enumerate(pg):
            for p, arr in enumerate(level):
                contrib[f"grid.l{l}.p{p}"] = arr
        for key, v in contrib.items():
            acc[key] = acc.get(key, 0.0) + v
        amb = O.pixel_decision_margins(out, cfg) < 1e-5
        for (ty, tx), (rows, xs, ys) in out["tiles"].items():
            if amb[ys[0]:ys[-1] + 1, xs[0]:xs[-1] + 1].any():
                bad[out["proj"]["source_index"][rows]] = True
    tv, tv_g = O.total_variation(field.planes, lam_tv)
    loss_ref += lam_tv * tv
    for l, level in enumerate(tv_g):
        for p, arr in enumerate(level):
            acc[f"grid.l{l}.p{p}"] = acc[f"grid.l{l}.p{p}"] + arr

    assert abs(loss - loss_ref) < 1e-5 * max(1.0, abs(loss_ref)), (loss, loss_ref)
    keep = ~bad
    assert keep.mean() > 0.5
    for key, ref in acc.items():
        got = step.grads[key].cpu().numpy().astype(np.float64).reshape(np.shape(ref))
        if np.shape(ref)[0] == k and key in ("positions", "rotations", "log_scales", "opacity_logits",
                                               "colors_raw", "sh_rest", "features"):
            got, ref = got[keep], np.asarray(ref)[keep]
        tol = max(1e-3 * np.abs(ref).max(), 1e-12)
        assert np.abs(got - ref).max() < tol, (key, np.abs(got - ref).max(), tol)

    # ---- Adam on the device's own gradients (stage injection) ----
    p1 = step.params.buffer.cpu().numpy().astype(np.float64)
    g0 = step.grads.buffer.cpu().numpy().astype(np.float64)
    p0 = p0.cpu().numpy().astype(np.float64)
    lrs = {key: s.lr_init for key, s in schedules.items()}  # iteration 0: lr_at_step(s, 0) == lr_init
    lrs["net"] = schedules["net"].lr_init * schedules["net"].delay_mult
    for (name, shape), off in zip(step.specs, step.params.offsets):
        n = int(np.prod(shape))
        lr = lrs["colors_raw"] if name == "sh_rest" else lrs[schedule_key(name)]
        ref, _, _, _ = O.adam_update(p0[off:off + n], g0[off:off + n], 0.0, 0.0, 0, lr, adam_eps(name))
        got = p1[off:off + n]
        assert np.abs(got - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), name
    assert step.iteration == 1


def test_checkpoint_round_trip_of_device_training_state(tmp_path):
    """save_train_state -> load_train_state into a fresh TrainStep restores
    parameters, Adam moments and step counts exactly; the next step of both
    agrees up to the backward's atomic-order noise (training.py:569-706
    semantics on device buffers)."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import checkpoint as ck
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.numerics import LrSchedule
    from paper_2503_06161_b200.train import TrainStep

    rng = np.random.default_rng(3)
    k, h, w, d = 800, 32, 48, 8
    a = random_cloud_arrays(rng, k, d, depth_range=(2.0, 4.0), xy=1.0)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    K = pinhole(h, w, 40.0)
    sched = {n: LrSchedule.constant(1e-3) for n in ("positions", "rotations", "log_scales", "opacity_logits",
                                                     "colors_raw", "features", "grid", "net")}

    def make():
        s = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                      h, w, fs.RasterConfig())
        return s.attach_optimizer(sched)

    batch = [(0.4, K, np.eye(4), torch.rand(h, w, 3, device="cuda"), torch.randn(h, w, d, device="cuda"))]
    s1 = make()
    for _ in range(2):
        s1.run(batch, check=True)
    p = str(tmp_path / "state.fs4c")
    ck.save_train_state(s1, p, meta={"meta.extent": 1.5})
    e = ck.load_entries(p)
    assert e["meta.iteration"] == 2 and e["adam.positions.step"] == 2 and e["cloud.positions"].dtype == np.float64
    s2 = make()
    ck.load_train_state(s2, p)
    assert torch.equal(s1.params.buffer, s2.params.buffer)
    assert torch.equal(s1.optimizer.m, s2.optimizer.m) and torch.equal(s1.optimizer.v, s2.optimizer.v)
    assert torch.equal(s1.optimizer.steps, s2.optimizer.steps) and s2.iteration == 2
    s1.run(batch, check=True)
    s2.run(batch, check=True)
    torch.cuda.synchronize()
    diff = (s1.params.buffer - s2.params.buffer).abs().max().item()
    assert diff < 1e-6, diff  # atomics in the backward: last-bit differences only


def test_density_control_inside_the_training_step():
    """TrainStep.track_stats + densify: the view-space statistics accumulate
    on device every step, and densify compacts parameters and Adam moments in
    the reference's row order (oracle density_control on the same pre-step
    state), keeps the network / plane state, and the next step runs at the
    new K."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.density import DensityControlConfig
    from paper_2503_06161_b200.numerics import LrSchedule
    from paper_2503_06161_b200.train import TrainStep

    rng = np.random.default_rng(11)
    k, h, w, d = 3000, 48, 64, 8
    a = random_cloud_arrays(rng, k, d, op_range=(0.001, 0.9), depth_range=(2.0, 4.0), xy=1.0,
                            ls_range=(0.005, 0.2), sh_degree=1)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    step = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                     h, w, fs.RasterConfig())
    step.attach_optimizer({n: LrSchedule.constant(1e-3) for n in ("positions", "rotations", "log_scales",
                                                                  "opacity_logits", "colors_raw", "features",
                                                                  "grid", "net")})
    step.track_stats()
    K = pinhole(h, w, 50.0)
    batch = [(0.3, K, np.eye(4), torch.rand(h, w, 3, device="cuda"), torch.randn(h, w, d, device="cuda"))]
    for _ in range(2):
        step.run(batch, check=True)
    torch.cuda.synchronize()
    counts = step.stats.count.cpu().numpy()
    assert counts.max() == 2 and (counts > 0).mean() > 0.5  # visible Gaussians counted once per step
    # oracle on the same pre-densify state
    names = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features")
    pre = {n: getattr(step.cloud, n).cpu().numpy().astype(np.float64) for n in names}
    pre["sh_rest"] = step.cloud.sh_rest.cpu().numpy().astype(np.float64)
    spec_names = [sn for sn, _ in step.specs]
    per = [n for n in ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "sh_rest", "features")]
    extras = []
    for n in per:
        i = spec_names.index(n)
        off, cnt = step.params.offsets[i], step.params.sizes[i]
        shape = tuple(step.params.views[n].shape)
        extras += [step.optimizer.m[off:off + cnt].cpu().numpy().astype(np.float64).reshape(shape),
                   step.optimizer.v[off:off + cnt].cpu().numpy().astype(np.float64).reshape(shape)]
    acc, cnt_ = step.stats.accum.cpu().numpy(), step.stats.count.cpu().numpy()
    thr = float(np.percentile(acc / np.maximum(cnt_, 1), 70))
    cfg = DensityControlConfig(grad_threshold=thr, percent_dense=0.05, prune_opacity=0.02)
    net_before = step.params["net.trunk.0.weight"].clone()
    rep = step.densify(cfg, 1.3, np.random.default_rng(5))
    cl = type("C", (), dict(pre))()
    zr = np.random.default_rng(5)
    ro, _, _, rex, rc = O.density_control(cl, acc, cnt_, thr, 0.05, 0.02, 1.6, 1.3,
                                          np.stack([zr.standard_normal((rep["split"], 3)) for _ in range(2)]),
                                          extras=extras)
    assert (rep["cloned"], rep["split"], rep["count"]) == (rc["clone"], rc["split"], len(ro["positions"]))
    assert rep["cloned"] > 0 and rep["split"] > 0
    for n in names + ("sh_rest",):
        got = getattr(step.cloud, n).cpu().numpy().astype(np.float64).reshape(ro[n].shape)
        tol = 1e-6 * max(1.0, np.abs(ro[n]).max()) if n in ("positions", "log_scales") else 0.0
        assert np.abs(got - ro[n]).max() <= tol, n
    for j, n in enumerate(per):
        i = [sn for sn, _ in step.specs].index(n)
        off, cnt = step.params.offsets[i], step.params.sizes[i]
        np.testing.assert_array_equal(step.optimizer.m[off:off + cnt].cpu().numpy().astype(np.float64),
                                      rex[2 * j].reshape(-1))
    assert torch.equal(step.params["net.trunk.0.weight"], net_before)
    assert not step.stats.accum.any() and len(step.stats.accum) == rep["count"]
    step.run(batch, check=True)  # the next step at the new K
    torch.cuda.synchronize()
    assert len(step.cloud) == rep["count"] and torch.isfinite(step.params.buffer).all()


def test_pairs_in_flight_match_serial_step():
    """TrainStep(lanes=L): pairs j, j+L, ... run on lane j's stream into the
    lane's gradient buffer (overwritten by its first pair, accumulated by the
    rest), summed before the reduce; view-space statistics serialised across
    lanes.  Same gradients, loss and statistics as the serial step up to fp32
    summation order."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.train import TrainStep

    rng = np.random.default_rng(5)
    k, h, w, d = 3000, 48, 64, 8
    a = random_cloud_arrays(rng, k, d, op_range=(0.05, 0.9), depth_range=(2.0, 4.0), xy=1.0,
                            ls_range=(0.01, 0.1), sh_degree=1)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    K = pinhole(h, w, 50.0)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    batch = [(float(t), K, rigid_T(rng), torch.rand(h, w, 3, device="cuda", generator=gen),
              torch.randn(h, w, d, device="cuda", generator=gen)) for t in np.linspace(0.05, 0.95, 7)]
    out = {}
    for lanes in (1, 2, 3):
        step = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field),
                         dv.DeviceNet.from_net(net), h, w, fs.RasterConfig(), lanes=lanes)
        step.track_stats()
        for _ in range(2):  # the second run reuses the lanes and their caches
            loss = float(step.run(batch, check=True).item())
        torch.cuda.synchronize()
        out[lanes] = (loss, step.grads.buffer.double().cpu().numpy(), step.stats.accum.cpu().numpy(),
                      step.stats.count.cpu().numpy())
    ref = out[1]
    scale = np.abs(ref[1]).max()
    for lanes in (2, 3):
        loss, g, acc, cnt = out[lanes]
        assert abs(loss - ref[0]) < 1e-9 * max(1.0, abs(ref[0]))
        assert np.abs(g - ref[1]).max() < 1e-5 * scale, (lanes, np.abs(g - ref[1]).max(), scale)
        np.testing.assert_array_equal(cnt, ref[3])
        np.testing.assert_allclose(acc, ref[2], rtol=1e-5, atol=1e-9)
