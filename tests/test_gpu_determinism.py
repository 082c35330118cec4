"""Deterministic backward mode (per-tile partials merged in
a fixed order; the reference tests bit-identical training and checkpoint
resume, test_training.py:225-235, 282-299):

* fs4d_render_bwd_deterministic -- ordered per-(pair, CTA) partials and a
  per-Gaussian gather -- and fs4d_deform_bwd_deterministic -- int64
  fixed-point HexPlane scatter -- give bitwise identical gradients run to run
  and agree with the atomic path to fp32 summation noise;
* TrainStep(deterministic=True) with three pairs in flight is bitwise
  reproducible (gradients, parameters, Adam state; the reported loss scalar
  to double rounding), and a save / load / continue of the device training
  state ends byte-identical to the unbroken run (FS4C files compared byte
  for byte).
"""

import numpy as np
import pytest

from conftest import has_gpu, pinhole, random_cloud_arrays, rigid_T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def _parts(seed, k=20_000, d=16):
    import paper_2503_06161_b200 as fs
    rng = np.random.default_rng(seed)
    a = random_cloud_arrays(rng, k, d, depth_range=(2.0, 4.0), xy=1.0, ls_range=(0.01, 0.06), sh_degree=3)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(16, 16, 16, 8), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    return cloud, field, net, rng


def test_render_and_deform_backward_bitwise_reproducible():
    import paper_2503_06161_b200 as fs
    cloud, field, net, rng = _parts(1)
    h, w = 96, 128
    fr = fs.CameraFrame(K=pinhole(h, w, 110.0), T=rigid_T(rng), time=0.3, image=np.zeros((h, w, 3)),
                        depth=np.zeros((h, w)), mask=np.ones((h, w), bool))
    snap, cache = fs.deform_with_cache(cloud, field, net, 0.3)
    out = fs.render(snap, fr, fs.RasterConfig())
    up = [rng.normal(size=(h, w, 3)), rng.normal(size=(h, w)), rng.normal(size=(h, w, 16)), rng.normal(size=(h, w))]
    g1 = fs.render_backward(snap, fr, out, *up, deterministic=True)
    g2 = fs.render_backward(snap, fr, out, *up, deterministic=True)
    ga = fs.render_backward(snap, fr, out, *up)
    fields = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features", "sh_rest")
    for f in fields:
        a, b, c = getattr(g1, f), getattr(g2, f), getattr(ga, f)
        assert np.array_equal(a, b), f
        assert np.abs(a - c).max() <= 1e-5 * max(1.0, np.abs(c).max()), f
    d1 = fs.deform_backward(cloud, field, net, cache, g1, deterministic=True)
    d2 = fs.deform_backward(cloud, field, net, cache, g1, deterministic=True)
    da = fs.deform_backward(cloud, field, net, cache, g1)
    assert np.array_equal(d1[0]["positions"], d2[0]["positions"])
    for key in d1[1]:
        assert np.array_equal(d1[1][key], d2[1][key]), key
    for l in range(2):
        for p in range(6):
            assert np.array_equal(d1[2][l][p], d2[2][l][p]), (l, p)
            ref = da[2][l][p]
            assert np.abs(d1[2][l][p] - ref).max() <= 1e-5 * max(1e-30, np.abs(ref).max()), (l, p)
    ref = da[0]["positions"]
    assert np.abs(d1[0]["positions"] - ref).max() <= 1e-5 * np.abs(ref).max()


def _train_step(cloud, field, net, h, w, deterministic=True):
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.numerics import LrSchedule
    from paper_2503_06161_b200.train import TrainStep
    s = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                  h, w, fs.RasterConfig(), lanes=3, deterministic=deterministic)
    return s.attach_optimizer({n: LrSchedule.constant(1e-3) for n in
                               ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features",
                                "grid", "net")})


def test_training_steps_and_checkpoint_resume_byte_identical(tmp_path):
    """The analogue of test_training.py:282-299 on the device: an unbroken
    run of 4 steps and a run saved after 2 steps, reloaded into a fresh
    TrainStep and continued for 2 steps end in byte-identical FS4C files."""
    import torch
    from paper_2503_06161_b200 import checkpoint as ck
    cloud, field, net, rng = _parts(2, k=15_000)
    h, w = 80, 112
    K = pinhole(h, w, 95.0)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    batch = [(float(t), K, rigid_T(rng), torch.rand(h, w, 3, device="cuda", generator=gen),
              torch.randn(h, w, 16, device="cuda", generator=gen)) for t in (0.1, 0.4, 0.6, 0.9, 0.7)]
    a = _train_step(cloud, field, net, h, w)
    b = _train_step(cloud, field, net, h, w)
    la = [float(a.run(batch, check=True).item()) for _ in range(2)]
    lb = [float(b.run(batch, check=True).item()) for _ in range(2)]
    # the reported loss scalar sums per-block double partials with atomics
    # (it is not model state): equal to double rounding
    assert np.allclose(la, lb, rtol=1e-12, atol=0)
    assert torch.equal(a.grads.buffer, b.grads.buffer) and torch.equal(a.params.buffer, b.params.buffer)
    mid = str(tmp_path / "mid.fs4c")
    ck.save_train_state(a, mid)
    for _ in range(2):
        a.run(batch, check=True)
    c = _train_step(cloud, field, net, h, w)
    ck.load_train_state(c, mid)
    for _ in range(2):
        c.run(batch, check=True)
    fa, fc = str(tmp_path / "a.fs4c"), str(tmp_path / "c.fs4c")
    ck.save_train_state(a, fa)
    ck.save_train_state(c, fc)
    assert open(fa, "rb").read() == open(fc, "rb").read()
    # the atomic (default) step agrees to fp32 summation noise
    d = _train_step(cloud, field, net, h, w, deterministic=False)
    d.run(batch, check=True)
    e = _train_step(cloud, field, net, h, w)
    e.run(batch, check=True)
    scale = e.grads.buffer.abs().max().item()
    assert (d.grads.buffer - e.grads.buffer).abs().max().item() <= 1e-5 * scale
