"""GPU parity of the training-step glue against the
reference's golden vectors and the float64 oracle: Adam (single array and the
multi-segment flat buffer), HexPlane TV loss/grad, bilinear resize + adjoint,
pointwise decoder fwd/bwd, the fused decoder feature loss, feature L1, and
the masked photometric L1.

Tolerances (fp32 arithmetic vs float64): 1e-6 relative to max(1, |x|max) for
elementwise maps (Adam, TV, resize, decoder); the sign() of an L1 term is a
discrete decision -- elements whose float64 residual is within 1e-5 of 0 are
margin-classified (their sign is taken from the device's own fp32 residual),
as SURVEY §8(c) does for the blend decisions."""

import numpy as np
import pytest

from conftest import has_gpu, load_golden
from oracle import fs4d_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


@pytest.fixture(scope="module")
def g():
    return load_golden("train_ops")


def close(a, b, rel=1e-6, what=""):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    tol = rel * max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    err = float(np.abs(a - b).max()) if a.size else 0.0
    assert err <= tol, f"{what}: max abs err {err:.3e} > {tol:.3e}"


# ---------------------------------------------------------------------------
# Adam
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("tag,eps", [("g", 1e-15), ("n", 1e-8)])
def test_adam_step_matches_reference_goldens(g, tag, eps):
    from paper_2503_06161_b200.numerics import AdamState, adam_step
    p = g[f"adam_{tag}_p0"]
    st = AdamState.for_param(p, eps=eps)
    for i in range(3):
        p = adam_step(p, g[f"adam_{tag}_g{i}"], st, 1e-3 * (i + 1))
        assert st.step_count == i + 1
        close(p, g[f"adam_{tag}_p{i + 1}"], 1e-6, f"param step {i}")
        close(st.m, g[f"adam_{tag}_m{i + 1}"], 1e-6, f"m step {i}")
        np.testing.assert_allclose(st.v, g[f"adam_{tag}_v{i + 1}"], rtol=1e-5, atol=1e-30)


def test_adam_step_errors_and_device_tensors():
    import torch
    from paper_2503_06161_b200.errors import ConfigurationError, NumericalError
    from paper_2503_06161_b200.numerics import AdamState, adam_step
    p = np.ones((4, 3))
    st = AdamState.for_param(p)
    with pytest.raises(ConfigurationError):
        adam_step(p, np.ones((4, 3)), st, 0.0)
    with pytest.raises(ConfigurationError):
        adam_step(p, np.ones((3, 4)), st, 1e-3)
    bad = np.ones((4, 3))
    bad[2, 1] = np.inf
    with pytest.raises(NumericalError, match="non-finite gradient"):
        adam_step(p, bad, st, 1e-3)
    assert st.step_count == 0 and not np.any(st.m)
    # CUDA tensors: in-place, no host round trip
    pt = torch.ones(5, device="cuda")
    st = AdamState.for_param(pt)
    out = adam_step(pt, torch.full((5,), 2.0, device="cuda"), st, 0.1)
    assert out is pt and st.step_count == 1
    np.testing.assert_allclose(pt.cpu().numpy(), 1.0 - 0.1, rtol=1e-6)


def test_flat_adam_segments_match_oracle():
    """Many segments with ragged sizes / offsets, per-segment lr and eps, three
    steps, then a non-finite gradient that must leave everything untouched."""
    import torch
    from paper_2503_06161_b200.errors import NumericalError
    from paper_2503_06161_b200.optim import FlatAdam, adam_eps

    rng = np.random.default_rng(3)
    specs = [("positions", (1001, 3)), ("rotations", (1001, 4)), ("opacity_logits", (1001,)),
             ("grid.l0.p0", (7, 9, 5)), ("net.trunk.0.weight", (13, 11)), ("net.trunk.0.bias", (13,)),
             ("decoder.bias", (1,)), ("features", (1001, 6))]
    sizes = [int(np.prod(s)) for _, s in specs]
    p0 = rng.normal(size=sum(sizes)).astype(np.float32)
    params = torch.tensor(p0, device="cuda")
    opt = FlatAdam(specs, params)
    ref = {n: [p0[o:o + s].astype(np.float64), 0.0, 0.0, 0]
           for (n, _), o, s in zip(specs, np.cumsum([0] + sizes[:-1]), sizes)}
    lrs = {"positions": 1.6e-4, "rotations": 1e-3, "opacity_logits": 5e-2, "grid": 1.6e-3, "net": 1.6e-4,
           "decoder": 1e-3, "features": 2.5e-3}
    for step in range(3):
        gr = (rng.normal(size=p0.size) * 10.0 ** rng.uniform(-5, 0, size=p0.size)).astype(np.float32)
        opt.step(torch.tensor(gr, device="cuda"), lrs)
        off = 0
        for (n, _), s in zip(specs, sizes):
            r = ref[n]
            lr = lrs[n] if n in lrs else lrs[n.split(".")[0]]
            r[0], r[1], r[2], r[3] = O.adam_update(r[0], gr[off:off + s].astype(np.float64), r[1], r[2], r[3], lr,
                                                   adam_eps(n))
            off += s
    opt.check()
    got = params.cpu().numpy()
    off = 0
    for (n, _), s in zip(specs, sizes):
        close(got[off:off + s], ref[n][0], 1e-6, n)
        off += s
    assert opt.steps.cpu().tolist() == [3] * len(specs)
    # non-finite gradient in the 5th segment: nothing moves, step counts stay
    snap = (params.clone(), opt.m.clone(), opt.v.clone())
    gr = torch.zeros_like(params)
    gr[sum(sizes[:4]) + 7] = float("nan")
    opt.step(gr, lrs)
    with pytest.raises(NumericalError, match="net.trunk.0.weight"):
        opt.check()
    assert torch.equal(params, snap[0]) and torch.equal(opt.m, snap[1]) and torch.equal(opt.v, snap[2])
    assert opt.steps.cpu().tolist() == [3] * len(specs)


# ---------------------------------------------------------------------------
# HexPlane TV
# ---------------------------------------------------------------------------
def test_tv_matches_reference_goldens(g):
    from paper_2503_06161_b200 import hexplane as hp

    class F:
        pass

    f = F()
    f.planes = [[g[f"tv_plane_{l}_{p}"] for p in range(6)] for l in range(2)]
    f.aabb = np.array([[-1.0, -1, -1], [1, 1, 1]])
    f.channels = f.planes[0][0].shape[2]
    assert hp.tv_loss(f) == pytest.approx(float(g["tv_loss"]), rel=1e-6)
    grads = hp.tv_backward(f, 0.37)
    for l in range(2):
        for p in range(6):
            close(grads[l][p], g[f"tv_grad_{l}_{p}"], 1e-6, f"tv grad {l},{p}")


def test_tv_accumulates_into_gradient_buffer():
    import torch
    from paper_2503_06161_b200.device import DeviceField
    from paper_2503_06161_b200.hexplane import tv_loss_grad_device
    rng = np.random.default_rng(5)
    planes = [[rng.normal(size=(ra, rb, 32)) for ra, rb in ((64, 64), (64, 64), (64, 25), (64, 64), (64, 25),
                                                            (64, 25))]]
    dev = DeviceField([[torch.tensor(p, dtype=torch.float32, device="cuda") for p in lv] for lv in planes],
                      np.array([[0.0, 0, 0], [1, 1, 1]]), 32)
    base = [[rng.normal(size=p.shape) for p in lv] for lv in planes]
    grads = DeviceField([[torch.tensor(b, dtype=torch.float32, device="cuda") for b in lv] for lv in base],
                        dev.aabb, 32)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    tv_loss_grad_device(dev, grads, 0.25, True, loss)
    ref_loss, ref_g = O.total_variation([[p.astype(np.float32).astype(np.float64) for p in lv] for lv in planes],
                                        0.25)
    assert float(loss.item()) == pytest.approx(0.25 * ref_loss, rel=1e-6)  # loss += scale * tv
    for p in range(6):
        close(grads.planes[0][p].cpu().numpy(), base[0][p] + ref_g[0][p], 1e-6, f"plane {p}")


# ---------------------------------------------------------------------------
# resize / decoder / feature loss
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("i", range(4))
def test_resize_and_adjoint_match_reference_goldens(g, i):
    from paper_2503_06161_b200 import semantic as sm
    img, dout = g[f"rs{i}_in"], g[f"rs{i}_dout"]
    close(sm.resize_bilinear(img, dout.shape[:2]), g[f"rs{i}_out"], 1e-6, "resize")
    close(sm.resize_bilinear_backward(dout, img.shape[:2]), g[f"rs{i}_din"], 1e-6, "adjoint")


def test_resize_render_resolution_adjoint_identity():
    """512x640x16 render-resolution map down to the 64x80 teacher grid and up:
    forward against the oracle, and <A x, y> == <x, A^T y>."""
    import torch
    from paper_2503_06161_b200 import semantic as sm
    rng = np.random.default_rng(9)
    for (hi, wi), (ho, wo) in (((512, 640), (64, 80)), ((64, 80), (512, 640))):
        x = torch.tensor(rng.normal(size=(hi, wi, 16)), dtype=torch.float32, device="cuda")
        y = torch.tensor(rng.normal(size=(ho, wo, 16)), dtype=torch.float32, device="cuda")
        ax = sm.resize_bilinear(x, (ho, wo))
        aty = sm.resize_bilinear_backward(y, (hi, wi))
        close(ax.cpu().numpy(), O.resize(x.cpu().numpy().astype(np.float64), (ho, wo)), 1e-6, "resize")
        lhs = float((ax.double() * y.double()).sum())
        rhs = float((x.double() * aty.double()).sum())
        assert lhs == pytest.approx(rhs, rel=1e-5)
        assert torch.equal(aty, sm.resize_bilinear_backward(y, (hi, wi)))  # gather: bitwise deterministic


def test_decoder_matches_reference_goldens(g):
    from paper_2503_06161_b200 import semantic as sm
    dec = sm.PointwiseDecoder(weight=g["dec_w"], bias=g["dec_b"])
    out, cache = sm.decode_features_with_cache(dec, g["dec_rendered"], g["dec_teacher"].shape[:2])
    close(out, g["dec_out"], 1e-6, "decoded")
    assert sm.feature_loss(out, g["dec_teacher"]) == pytest.approx(float(g["dec_loss"]), rel=1e-6)
    d_dec = 0.7 * sm.feature_loss_backward(out, g["dec_teacher"])
    dr, dw, db = sm.decode_features_backward(dec, cache, d_dec)
    close(dr, g["dec_d_rendered"], 1e-6, "d_rendered")
    close(dw, g["dec_dw"], 1e-6, "d_weight")
    close(db, g["dec_db"], 1e-6, "d_bias")


def _fused_case(rng, hi, wi, n, ho, wo, ct, lam):
    import torch
    from paper_2503_06161_b200 import semantic as sm
    f = dict(dtype=torch.float32, device="cuda")
    rendered = torch.tensor(rng.normal(size=(hi, wi, n)), **f)
    teacher = torch.tensor(rng.normal(size=(ho, wo, ct)), **f)
    w = torch.tensor(rng.uniform(-1, 1, size=(ct, n)) * np.sqrt(6.0 / n), **f)
    b = torch.tensor(rng.normal(size=ct) * 0.1, **f)
    d_r = torch.empty_like(rendered)
    dw, db = torch.full((ct, n), 0.5, **f), torch.full((ct,), 0.25, **f)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    sm.DecoderLoss()(w, b, rendered, teacher, lam, d_r, dw, db, loss, accumulate=True)
    # oracle, with margin-classified signs taken from the device's decoded map
    dev_out = sm.decode_features(sm.PointwiseDecoder(w, b), rendered, (ho, wo)).cpu().numpy()
    W, B, R, Tt = (x.cpu().numpy().astype(np.float64) for x in (w, b, rendered, teacher))
    out, resized = O.decoder_forward(W, B, R, (ho, wo))
    diff = out - Tt
    amb = np.abs(diff) < 1e-5
    sign = np.where(amb, np.sign(dev_out - Tt), np.sign(diff))
    d_out = lam * sign / (ho * wo)
    ref_loss = lam * np.abs(diff).sum() / (ho * wo)
    ref_dr, ref_dw, ref_db = O.decoder_backward(W, resized, (hi, wi), d_out)
    assert float(loss.item()) == pytest.approx(ref_loss, rel=1e-5)
    close(d_r.cpu().numpy(), ref_dr, 1e-5, "d_rendered")
    close(dw.cpu().numpy(), 0.5 + ref_dw, 1e-5, "d_weight")
    close(db.cpu().numpy(), 0.25 + ref_db, 1e-5, "d_bias")
    return int(amb.sum())


def test_fused_decoder_feature_loss_matches_oracle():
    rng = np.random.default_rng(11)
    n_amb = _fused_case(rng, 128, 160, 16, 64, 80, 32, 0.8)   # render 4x teacher grid
    n_amb += _fused_case(rng, 40, 56, 8, 40, 56, 24, 1.0)     # same resolution
    n_amb += _fused_case(rng, 33, 47, 5, 70, 29, 3, 0.3)      # ragged, up in y, down in x
    assert n_amb < 20


def test_decoder_rejects_bad_shapes():
    from paper_2503_06161_b200 import semantic as sm
    from paper_2503_06161_b200.errors import ConfigurationError
    dec = sm.PointwiseDecoder(weight=np.ones((4, 3)), bias=np.zeros(4))
    with pytest.raises(ConfigurationError):
        sm.decode_features(dec, np.ones((5, 5, 2)), (3, 3))
    with pytest.raises(ConfigurationError):
        sm.feature_loss(np.ones((2, 2, 3)), np.ones((2, 3, 3)))


# ---------------------------------------------------------------------------
# photometric L1
# ---------------------------------------------------------------------------
def _photometric_dev(color, image, mask, depth, depth_t, alpha, lam_rgb, lam_d):
    import torch
    from paper_2503_06161_b200.train import photometric_loss_grad
    f = dict(dtype=torch.float32, device="cuda")
    t = lambda x: torch.tensor(x, **f)  # noqa: E731
    dC = torch.empty(color.shape, **f)
    dD = torch.empty(depth.shape, **f)
    terms = photometric_loss_grad(t(color), t(image), torch.tensor(mask, device="cuda"), t(depth), t(depth_t),
                                  t(alpha), lam_rgb, lam_d, dC, dD)
    return terms.cpu().numpy(), dC.cpu().numpy(), dD.cpu().numpy()


def test_photometric_matches_reference_goldens(g):
    terms, dC, dD = _photometric_dev(g["ph_color"], g["ph_image"], g["ph_mask"], g["ph_depth"], g["ph_depth_t"],
                                     g["ph_alpha"], 0.8, 0.3)
    assert terms[0] == pytest.approx(float(g["ph_rgb"]), rel=1e-6)
    assert terms[1] == pytest.approx(float(g["ph_dterm"]), rel=1e-6)
    close(dC, g["ph_dC"], 1e-6, "dC")
    close(dD, g["ph_dD"], 1e-6, "dD")


def test_photometric_render_resolution_and_empty_mask():
    rng = np.random.default_rng(12)
    h, w = 512, 640
    c, img = rng.uniform(size=(h, w, 3)), rng.uniform(size=(h, w, 3))
    d, dt, a = rng.uniform(1, 3, (h, w)), rng.uniform(1, 3, (h, w)), rng.uniform(size=(h, w))
    f32 = lambda x: x.astype(np.float32).astype(np.float64)  # noqa: E731
    c, img, d, dt, a = map(f32, (c, img, d, dt, a))
    mask = rng.uniform(size=(h, w)) > 0.1
    terms, dC, dD = _photometric_dev(c, img, mask, d, dt, a, 1.0, 0.5)
    rgb, dterm, rC, rD = O.photometric(c, img, mask, d, dt, a, 1.0, 0.5)
    assert terms[0] == pytest.approx(rgb, rel=1e-6) and terms[1] == pytest.approx(dterm, rel=1e-6)
    close(dC, rC, 1e-6, "dC")
    close(dD, rD, 1e-6, "dD")
    terms, dC, dD = _photometric_dev(c, img, np.zeros((h, w), bool), d, dt, a, 1.0, 0.5)
    assert terms[0] == 0.0 and terms[1] == 0.0 and not dC.any() and not dD.any()
