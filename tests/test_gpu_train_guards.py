"""Error handling and per-array stepping of the device training step
(train.TrainStep, optim.FlatAdam):

* an asynchronous step (check=False) whose render overflows the tile-pair
  buffer or sees a non-finite snapshot skips its Adam update ON THE DEVICE
  (fs4d_status_merge gates fs4d_adam_step) and the error is raised by the
  next run() / sync(), with the pair buffer already grown;
* the Adam status block is reset every step, so one bad step does not freeze
  the optimizer;
* only the arrays the reference would have in its gradient dict are stepped
  (training.py:509-531): without feature supervision `features` and
  decoder.* keep their parameters, moments and step counts.
"""

import numpy as np
import pytest

from conftest import has_gpu, pinhole, random_cloud_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


SCHED_KEYS = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features", "grid", "net",
              "decoder")


def _parts(seed=0, k=2000, d=8):
    import paper_2503_06161_b200 as fs
    rng = np.random.default_rng(seed)
    a = random_cloud_arrays(rng, k, d, depth_range=(2.0, 4.0), xy=1.0, ls_range=(0.02, 0.12))
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    return cloud, field, net


def _step(cloud, field, net, h, w, **kw):
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.numerics import LrSchedule
    from paper_2503_06161_b200.train import TrainStep
    s = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                  h, w, fs.RasterConfig(), **kw)
    return s.attach_optimizer({n: LrSchedule.constant(1e-3) for n in SCHED_KEYS})


def test_pair_overflow_skips_the_step_on_device_and_raises_next_run():
    import torch
    from paper_2503_06161_b200._native import CapacityError
    cloud, field, net = _parts()
    h, w, d = 48, 64, 8
    step = _step(cloud, field, net, h, w, lanes=1)
    batch = [(0.4, pinhole(h, w, 50.0), np.eye(4), torch.rand(h, w, 3, device="cuda"),
              torch.randn(h, w, d, device="cuda"))]
    step.run(batch, check=True)  # sizes the pair buffer
    torch.cuda.synchronize()
    ln = step._lanes[0]
    ln.renderer.cap = 64        # far too small: the next async step overflows
    before = step.params.buffer.clone()
    m_before = step.optimizer.m.clone()
    steps_before = step.optimizer.steps.clone()
    step.run(batch)             # check=False: no host sync, no exception yet
    assert step.iteration == 2
    torch.cuda.synchronize()    # (the next run() raises as soon as the step's status copy has landed)
    with pytest.raises(CapacityError, match="skipped"):
        step.run(batch)
    # the failed step never touched the parameters, moments or step counts
    assert torch.equal(step.params.buffer, before) and torch.equal(step.optimizer.m, m_before)
    assert torch.equal(step.optimizer.steps, steps_before)
    assert step.iteration == 1
    assert ln.renderer.cap > 64  # grown past the overflowing step's pair count before raising
    step.run(batch, check=True)  # the same batch now succeeds
    assert step.iteration == 2 and not torch.equal(step.params.buffer, before)


def test_non_finite_snapshot_skips_the_step():
    import torch
    from paper_2503_06161_b200.errors import NumericalError
    cloud, field, net = _parts(1)
    h, w, d = 32, 48, 8
    step = _step(cloud, field, net, h, w, lanes=2)
    batch = [(t, pinhole(h, w, 40.0), np.eye(4), torch.rand(h, w, 3, device="cuda"),
              torch.randn(h, w, d, device="cuda")) for t in (0.2, 0.6)]
    step.run(batch, check=True)
    step.params["opacity_logits"][7] = float("nan")
    before = step.params.buffer.clone()
    step.run(batch)
    with pytest.raises(NumericalError, match="opacity_logits"):
        step.sync()
    assert torch.equal(torch.nan_to_num(step.params.buffer), torch.nan_to_num(before))
    assert step.iteration == 1


def test_adam_status_resets_every_step():
    """A non-finite gradient aborts that step only; the next step applies."""
    import torch
    from paper_2503_06161_b200.errors import NumericalError
    from paper_2503_06161_b200.optim import FlatAdam
    specs = [("a", (1000,)), ("net.b", (37,))]
    p = torch.zeros(1056, device="cuda")
    opt = FlatAdam(specs, p, offsets=[0, 1008])
    g = torch.ones(1056, device="cuda")
    g[1010] = float("inf")
    opt.step(g, {"a": 0.1, "net": 0.1})
    with pytest.raises(NumericalError, match="net.b"):
        opt.check()
    assert not p.any() and not opt.steps.any()
    g[1010] = 1.0
    opt.step(g, {"a": 0.1, "net": 0.1})
    opt.check()
    assert opt.steps.tolist() == [1, 1]
    assert torch.allclose(p[:1000], torch.full((1000,), -0.1, device="cuda"))


def test_only_supervised_arrays_are_stepped():
    """Decoder loss mode with no teacher in the batch: like the reference's
    fine stage without feature supervision (training.py:513-515, 531), the
    features and the decoder keep parameters, moments and step counts; every
    other array steps."""
    import torch
    cloud, field, net = _parts(2)
    h, w, d, ct = 32, 48, 8, 6
    dec = (torch.randn(ct, d, device="cuda") * 0.3, torch.zeros(ct, device="cuda"))
    step = _step(cloud, field, net, h, w, loss_mode="decoder", decoder=dec, lanes=1)
    batch = [(0.5, pinhole(h, w, 40.0), np.eye(4), torch.rand(h, w, 3, device="cuda"), None)]
    before = {n: step.params[n].clone() for n in ("features", "decoder.weight", "positions")}
    step.run(batch, check=True)
    names = [n for n, _ in step.specs]
    steps = dict(zip(names, step.optimizer.steps.tolist()))
    assert steps["features"] == 0 and steps["decoder.weight"] == 0 and steps["decoder.bias"] == 0
    assert steps["positions"] == 1 and steps["grid.l0.p0"] == 1 and steps["net.trunk.0.weight"] == 1
    assert torch.equal(step.params["features"], before["features"])
    assert torch.equal(step.params["decoder.weight"], before["decoder.weight"])
    assert not torch.equal(step.params["positions"], before["positions"])
    # with a teacher map the features and the decoder step too
    teacher = torch.randn(h // 2, w // 2, ct, device="cuda")
    step.run([(0.5, pinhole(h, w, 40.0), np.eye(4), torch.rand(h, w, 3, device="cuda"), teacher)], check=True)
    steps = dict(zip(names, step.optimizer.steps.tolist()))
    assert steps["features"] == 1 and steps["decoder.weight"] == 1 and steps["positions"] == 2
