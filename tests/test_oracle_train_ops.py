"""Pin the oracle's training-glue restatements (Adam, LR schedule, HexPlane TV,
bilinear resize + adjoint, pointwise decoder, feature L1, masked photometric
L1) to golden vectors produced by the reference itself
(tests/golden/make_golden.py train_ops_case).  Plus the host-side mirrors
that need no GPU (LrSchedule / lr_at_step, Adam segment naming).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fs4d_oracle as O


@pytest.fixture(scope="module")
def g():
    return load_golden("train_ops")


@pytest.mark.parametrize("tag,eps", [("g", 1e-15), ("n", 1e-8)])
def test_oracle_adam_three_steps(g, tag, eps):
    p, m, v, step = g[f"adam_{tag}_p0"], 0.0, 0.0, 0
    for i in range(3):
        p, m, v, step = O.adam_update(p, g[f"adam_{tag}_g{i}"], m, v, step, 1e-3 * (i + 1), eps)
        np.testing.assert_allclose(p, g[f"adam_{tag}_p{i + 1}"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(m, g[f"adam_{tag}_m{i + 1}"], rtol=1e-13, atol=0)
        np.testing.assert_allclose(v, g[f"adam_{tag}_v{i + 1}"], rtol=1e-13, atol=0)


def test_oracle_adam_rejects():
    with pytest.raises(O.OracleError):
        O.adam_update(np.zeros(3), np.array([0.0, np.nan, 1.0]), 0.0, 0.0, 0, 1e-3, 1e-8)
    with pytest.raises(O.OracleError):
        O.adam_update(np.zeros(3), np.zeros(3), 0.0, 0.0, 0, 0.0, 1e-8)


def test_oracle_and_host_lr_schedule(g):
    from paper_2503_06161_b200.numerics import LrSchedule, lr_at_step
    for i, t in enumerate(g["lr_steps"]):
        t = int(t)
        assert O.learning_rate(1.6e-4, 1.6e-6, 20000, t) == pytest.approx(g["lr_decay"][i], rel=1e-13)
        assert O.learning_rate(1.6e-3, 1.6e-4, 20000, t, 0.01, 500) == pytest.approx(g["lr_delay"][i], rel=1e-13)
        # the product's host mirror is the reference formula itself: bit-exact
        assert lr_at_step(LrSchedule(1.6e-4, 1.6e-6, 20000), t) == g["lr_decay"][i]
        assert lr_at_step(LrSchedule(1.6e-3, 1.6e-4, 20000, 0.01, 500), t) == g["lr_delay"][i]


def test_host_schedule_validation():
    from paper_2503_06161_b200.errors import ConfigurationError
    from paper_2503_06161_b200.numerics import LrSchedule, lr_at_step
    with pytest.raises(ConfigurationError):
        LrSchedule(0.0, 1.0, 10)
    with pytest.raises(ConfigurationError):
        LrSchedule(1.0, 1.0, 0)
    with pytest.raises(ConfigurationError):
        LrSchedule(1.0, 1.0, 10, delay_mult=0.0)
    with pytest.raises(ConfigurationError):
        lr_at_step(LrSchedule.constant(1.0), -1)


def test_adam_segment_naming():
    from paper_2503_06161_b200.optim import adam_eps, schedule_key
    assert adam_eps("positions") == 1e-15 and adam_eps("grid.l0.p1") == 1e-8
    assert adam_eps("net.trunk.0.weight") == 1e-8 and adam_eps("decoder.bias") == 1e-8
    assert schedule_key("grid.l1.p5") == "grid" and schedule_key("net.ext.scale.1.bias") == "net"
    assert schedule_key("decoder.weight") == "decoder" and schedule_key("log_scales") == "log_scales"


def _planes(g, prefix):
    return [[g[f"{prefix}_{l}_{p}"] for p in range(6)] for l in range(2)]


def test_oracle_tv(g):
    loss, grads = O.total_variation(_planes(g, "tv_plane"), 0.37)
    assert loss == pytest.approx(float(g["tv_loss"]), rel=1e-13)
    for l, level in enumerate(grads):
        for p, gr in enumerate(level):
            np.testing.assert_allclose(gr, g[f"tv_grad_{l}_{p}"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("i", range(4))
def test_oracle_resize_and_adjoint(g, i):
    img, dout = g[f"rs{i}_in"], g[f"rs{i}_dout"]
    np.testing.assert_allclose(O.resize(img, dout.shape[:2]), g[f"rs{i}_out"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.resize_adjoint(dout, img.shape[:2]), g[f"rs{i}_din"], rtol=0, atol=1e-13)


def test_oracle_decoder_and_feature_loss(g):
    out, resized = O.decoder_forward(g["dec_w"], g["dec_b"], g["dec_rendered"], g["dec_teacher"].shape[:2])
    np.testing.assert_allclose(out, g["dec_out"], rtol=0, atol=1e-13)
    loss, d_dec = O.l1_mean_pixels(out, g["dec_teacher"])
    assert loss == pytest.approx(float(g["dec_loss"]), rel=1e-13)
    dr, dw, db = O.decoder_backward(g["dec_w"], resized, g["dec_rendered"].shape[:2], 0.7 * d_dec)
    np.testing.assert_allclose(dr, g["dec_d_rendered"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(dw, g["dec_dw"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(db, g["dec_db"], rtol=0, atol=1e-13)


def test_oracle_photometric(g):
    rgb, dterm, dC, dD = O.photometric(g["ph_color"], g["ph_image"], g["ph_mask"], g["ph_depth"], g["ph_depth_t"],
                                       g["ph_alpha"], 0.8, 0.3)
    assert rgb == pytest.approx(float(g["ph_rgb"]), rel=1e-13)
    assert dterm == pytest.approx(float(g["ph_dterm"]), rel=1e-13)
    np.testing.assert_allclose(dC, g["ph_dC"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(dD, g["ph_dD"], rtol=0, atol=1e-15)
