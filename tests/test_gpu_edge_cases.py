"""GPU edge cases the reference tests (test_rasterizer.py) exercise: closed
forms, culls, empty/ragged inputs, error taxonomy, capacity retry, and
size-independent properties at BASELINE sizes."""

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


def fs():
    import paper_2503_06161_b200 as m
    return m


def frame(size=None, h=None, w=None, focal=None, T=None):
    h = h or size
    w = w or size
    focal = focal if focal is not None else 1.1 * w
    return fs().CameraFrame(K=pinhole(h, w, focal), T=np.eye(4) if T is None else T, time=0.0,
                            image=np.zeros((h, w, 3)), depth=np.zeros((h, w)), mask=np.ones((h, w), bool))


def lone(position, opacity, color, scale=0.5, feature=None):
    feature = np.zeros(2) if feature is None else feature
    return fs().GaussianCloud(positions=np.asarray([position], float), rotations=np.array([[1.0, 0, 0, 0]]),
                              log_scales=np.log(np.full((1, 3), scale)),
                              opacity_logits=np.asarray([float(fs().logit(opacity))]),
                              colors_raw=np.asarray([color], float), features=np.asarray([feature], float))


def stack(*clouds):
    return fs().GaussianCloud(*(np.concatenate([getattr(c, f) for c in clouds]) for f in
                                ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw",
                                 "features")))


def test_on_axis_projection_closed_form():
    f, d, s = 40.0, 4.0, 0.5
    proj = fs().project(lone([0, 0, d], 0.5, [0.5] * 3, scale=s), frame(32, focal=f), fs().RasterConfig())
    assert len(proj) == 1
    np.testing.assert_allclose(proj.cov2d[0], (f * s / d) ** 2 * np.eye(2) + 0.3 * np.eye(2), rtol=1e-6)
    np.testing.assert_allclose(proj.mean2d[0], [15.5, 15.5], atol=1e-5)


def test_behind_camera_and_offscreen_culled():
    assert len(fs().project(lone([0, 0, -2.0], 0.5, [0.5] * 3), frame(16), fs().RasterConfig())) == 0
    assert len(fs().project(lone([50.0, 0, 2.0], 0.5, [0.5] * 3, scale=0.01), frame(16),
                            fs().RasterConfig())) == 0


def test_depth_sort_stable_with_ties():
    cloud = stack(lone([0.3, 0, 3.0], 0.4, [0.9, 0.1, 0.1]), lone([-0.3, 0, 3.0], 0.4, [0.1, 0.9, 0.1]),
                  lone([0.0, 0, 2.0], 0.4, [0.1, 0.1, 0.9]))
    proj = fs().project(cloud, frame(32), fs().RasterConfig())
    assert proj.source_index.tolist() == [2, 0, 1]


def test_single_and_stacked_blend_closed_forms():
    out = fs().render(lone([0, 0, 3.0], 0.6, [1.0, 0, 0], scale=0.8), frame(17),
                      fs().RasterConfig(with_features=False))
    np.testing.assert_allclose(out.color[8, 8], [0.6, 0, 0], atol=1e-6)
    assert out.alpha[8, 8] == pytest.approx(0.6, abs=1e-6)
    assert out.depth[8, 8] == pytest.approx(1.8, abs=1e-5)
    c1, c2 = np.array([1.0, 0, 0]), np.array([0, 1.0, 0])
    out = fs().render(stack(lone([0, 0, 2.0], 0.5, c1, 0.8), lone([0, 0, 4.0], 0.5, c2, 1.6)), frame(17),
                      fs().RasterConfig(with_features=False))
    np.testing.assert_allclose(out.color[8, 8], 0.5 * c1 + 0.25 * c2, atol=1e-6)
    src, alphas, weights = out.pixel_record(8, 8)
    assert src.tolist() == [0, 1]


def test_background_and_feature_saturation():
    bg = np.array([0.2, 0.4, 0.6])
    out = fs().render(lone([0, 0, 3.0], 0.6, [1.0, 0, 0], scale=0.8), frame(17),
                      fs().RasterConfig(background=bg, with_features=False))
    np.testing.assert_allclose(out.color[8, 8], [0.6, 0, 0] + 0.4 * bg, atol=1e-6)
    z = np.array([0.7, -1.3, 2.0])
    parts = [lone([0, 0, 2.0 + 0.2 * i], 0.985, [0.5] * 3, scale=1.2, feature=z) for i in range(4)]
    out = fs().render(stack(*parts), frame(17), fs().RasterConfig())
    assert 1 - out.alpha[8, 8] < 1e-4
    np.testing.assert_allclose(out.feature[8, 8], z, atol=1e-3)


def test_empty_cloud_and_all_culled():
    rng = np.random.default_rng(0)
    a = random_cloud_arrays(rng, 0, 4)
    out = fs().render(fs().GaussianCloud(**{k: v for k, v in a.items()}), frame(20), fs().RasterConfig())
    assert np.all(out.alpha == 0) and np.all(out.color == 0)
    a = random_cloud_arrays(rng, 50, 4)
    a["positions"][:, 2] = -3.0
    out = fs().render(fs().GaussianCloud(**{k: v for k, v in a.items()}), frame(20), fs().RasterConfig())
    assert np.all(out.alpha == 0)
    g = fs().render_backward(fs().GaussianCloud(**{k: v for k, v in a.items()}), frame(20), out,
                             np.ones((20, 20, 3)))
    assert np.all(g.positions == 0) and g.viewspace_index.size == 0


def test_errors_map_to_reference_taxonomy():
    c = lone([0, 0, 3.0], 0.5, [0.5] * 3)
    c.positions[0, 1] = np.nan
    with pytest.raises(fs().NumericalError, match="0"):
        fs().render(c, frame(16), fs().RasterConfig())
    c = lone([0, 0, 3.0], 0.5, [0.5] * 3)
    c.rotations[:] = 0.0
    with pytest.raises(fs().DegenerateRotationError):
        fs().render(c, frame(16), fs().RasterConfig())
    fr = frame(16)
    fr.K[0, 1] = 0.5
    with pytest.raises(fs().DataError):
        fs().render(lone([0, 0, 3.0], 0.5, [0.5] * 3), fr, fs().RasterConfig())
    rng = np.random.default_rng(3)
    a = random_cloud_arrays(rng, 6, 4)
    b = random_cloud_arrays(rng, 7, 4)
    out = fs().render(fs().GaussianCloud(**a), frame(16), fs().RasterConfig())
    with pytest.raises(fs().ContractViolation):
        fs().render_backward(fs().GaussianCloud(**b), frame(16), out)


def test_capacity_overflow_retries_without_changing_result():
    from paper_2503_06161_b200.device import DeviceCloud, Renderer
    rng = np.random.default_rng(5)
    a = random_cloud_arrays(rng, 3000, 8, ls_range=(0.05, 0.2))
    cloud = DeviceCloud.from_cloud(fs().GaussianCloud(**a))
    K = pinhole(64, 96, 80.0)
    cfg = fs().RasterConfig()
    big = Renderer(pair_capacity=10_000_000)
    ref, rec = big.forward(cloud, K, np.eye(4), 64, 96, cfg)
    small = Renderer(pair_capacity=64)
    got, rec2 = small.forward(cloud, K, np.eye(4), 64, 96, cfg)
    assert small.cap > 64 and rec2.n_pairs == rec.n_pairs
    for key in ("color", "feature", "alpha", "n_contrib"):
        assert bool((ref[key] == got[key]).all())


@pytest.mark.parametrize("nf", [0, 3, 13, 40])
def test_feature_widths_and_ragged_sizes(nf):
    """D = 0 (with_features off), odd D, D > 32 (chunked blend); 33x47 ragged tiles."""
    from oracle import fs4d_oracle as O
    rng = np.random.default_rng(nf)
    a = random_cloud_arrays(rng, 400, nf, ls_range=(0.03, 0.15))
    K = pinhole(33, 47, 40.0)
    fr = fs().CameraFrame(K=K, T=np.eye(4), time=0.0, image=np.zeros((33, 47, 3)), depth=np.zeros((33, 47)),
                          mask=np.ones((33, 47), bool))
    cfg = fs().RasterConfig(with_features=nf != 13)
    out = fs().render(fs().GaussianCloud(**a), fr, cfg)
    ref = O.render(type("C", (), a)(), K, np.eye(4), 33, 47, O.RasterParams(with_features=cfg.with_features))
    amb = O.pixel_decision_margins(ref, O.RasterParams()) < 1e-5
    for key in ("color", "feature", "alpha", "depth"):
        d = np.abs(getattr(out, key) - ref[key])
        if d.size:
            d = d.reshape(33, 47, -1).max(axis=2)
            assert d[~amb].max() < 1e-4, key


def test_size_independent_properties_at_config1_size():
    """At the 640x512 / 200k headline size: linearity in a shared feature,
    conservation (alpha + T = 1), colour bound, determinism of the device path."""
    import torch
    from paper_2503_06161_b200.device import DeviceCloud, Renderer
    rng = np.random.default_rng(9)
    k, h, w = 200_000, 512, 640
    a = random_cloud_arrays(rng, k, 16, op_range=(0.05, 0.95), depth_range=(3.0, 6.0), xy=1.0,
                            ls_range=(np.exp(-5.0), np.exp(-3.0)))
    zstar = np.linspace(-1.0, 1.0, 16)
    a["features"] = np.tile(zstar, (k, 1))
    a["colors_raw"] = np.tile([0.25, 0.5, 0.75], (k, 1))
    cloud = DeviceCloud.from_cloud(fs().GaussianCloud(**a))
    r = Renderer()
    K = pinhole(h, w, 560.0)
    img, rec = r.forward(cloud, K, np.eye(4), h, w, fs().RasterConfig())
    alpha = img["alpha"].cpu().numpy()
    feat = img["feature"].cpu().numpy()
    col = img["color"].cpu().numpy()
    assert alpha.min() >= 0 and alpha.max() <= 1
    np.testing.assert_allclose(feat, alpha[:, :, None] * zstar[None, None, :], atol=2e-5)
    np.testing.assert_allclose(col, alpha[:, :, None] * np.array([0.25, 0.5, 0.75]), atol=2e-5)
    img2, _ = r.forward(cloud, K, np.eye(4), h, w, fs().RasterConfig())
    for key in img:
        assert torch.equal(img[key], img2[key])
    assert rec.n_visible > 0.95 * k


def test_size_independent_properties_at_config3_size():
    """configs[3] (SCARED-shaped): 500k Gaussians, 1280x1024, fx=fy=1100, SH3,
    D=32 -- long tile lists and the 32-channel feature registers.  Linearity
    in a shared feature and colour, conservation, determinism, and the pair
    count / visible set of the device binning against the float64 oracle's
    projection + binning of the same scene."""
    import torch
    from oracle import fs4d_oracle as O
    from paper_2503_06161_b200.device import DeviceCloud, Renderer
    rng = np.random.default_rng(13)
    k, h, w, d = 500_000, 1024, 1280, 32
    a = random_cloud_arrays(rng, k, d, op_range=(0.05, 0.95), depth_range=(3.0, 6.0), xy=1.0,
                            ls_range=(np.exp(-5.0), np.exp(-3.0)), sh_degree=3)
    zstar = np.linspace(-1.0, 1.0, d)
    a["features"] = np.tile(zstar, (k, 1))
    a["colors_raw"] = np.tile([0.25, 0.5, 0.75], (k, 1))
    a["sh_rest"] = np.zeros_like(a["sh_rest"])  # colour = clip(DC) everywhere -> linearity holds
    cloud_np = fs().GaussianCloud(**a)
    cloud = DeviceCloud.from_cloud(cloud_np)
    r = Renderer()
    K = pinhole(h, w, 1100.0)
    img, rec = r.forward(cloud, K, np.eye(4), h, w, fs().RasterConfig())
    alpha = img["alpha"].cpu().numpy()
    assert alpha.min() >= 0 and alpha.max() <= 1
    np.testing.assert_allclose(img["feature"].cpu().numpy(), alpha[:, :, None] * zstar[None, None, :], atol=3e-5)
    np.testing.assert_allclose(img["color"].cpu().numpy(), alpha[:, :, None] * np.array([0.25, 0.5, 0.75]),
                               atol=3e-5)
    img2, _ = r.forward(cloud, K, np.eye(4), h, w, fs().RasterConfig())
    for key in img:
        assert torch.equal(img[key], img2[key])
    proj = O.project(cloud_np, K, np.eye(4), h, w, O.RasterParams())
    lists = O.bin_tiles(proj, h, w, 16)
    n_pairs = sum(c.size for row in lists for c in row)
    assert rec.n_visible == len(proj["source_index"])
    assert rec.n_pairs == n_pairs


def test_sequence_renderer_frames_in_flight_match_serial_frames():
    """configs[2]-style sequence with frames in flight on two streams (and a
    model replica per pipeline) gives exactly the frames a single pipeline
    renders one at a time."""
    import torch
    from paper_2503_06161_b200 import device as dv
    rng = np.random.default_rng(21)
    k, h, w, d = 20_000, 128, 160, 8
    a = random_cloud_arrays(rng, k, d, depth_range=(2.0, 4.0), xy=1.0)
    cloud_np = fs().GaussianCloud(**a)
    field_np = fs().HexPlaneField(fs().HexPlaneConfig(levels=(1, 2), base_resolution=(16, 16, 16, 5), out_dim=64),
                                  fs().scene_aabb(cloud_np), rng, init="uniform")
    net_np = fs().DeformationNet(64, fs().DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                                 head_init="xavier")
    c, f, n = dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np), dv.DeviceNet.from_net(net_np)
    K = pinhole(h, w, 150.0)
    ts = [i / 11.0 for i in range(12)]
    single = dv.FramePipeline(c, f, n, h, w, fs().RasterConfig())
    ref = []
    for t in ts:
        single.run(t, K, np.eye(4), check=True)
        ref.append({key: v.clone() for key, v in single.images.items()})
    seq = dv.SequenceRenderer(c, f, n, h, w, fs().RasterConfig(), pipelines=4, streams=2, replicas=4)
    seq.warm(0.0, K, np.eye(4))
    outs = []
    for r0 in range(0, len(ts), 4):  # one round = one frame per pipeline, copied out after the round
        seq.run(ts[r0:r0 + 4], K, np.eye(4))
        torch.cuda.synchronize()
        for p in range(4):
            outs.append({key: v.clone() for key, v in seq.pipes[p].images.items()})
    seq.raise_if_error()
    for got, exp in zip(outs, ref):
        for key in exp:
            assert torch.equal(got[key], exp[key]), key


@pytest.mark.parametrize("case", ["planes", "few_ties"])
def test_tile_sort_clustered_depths_and_fp32_ties(case):
    """Per-tile sort edge cases (binning.cu), seen by a camera tilted by
    1e-7 rad so that equal fp32 depth keys still differ by ~1e-8 in fp64:
    'planes' -- 3000 Gaussians on three depth planes only: the keys collide in
    large runs, the bucket map degenerates and the radix fallback runs;
    'few_ties' -- depths spread over [3, 6] except 40 Gaussians at exactly
    4.0: the bucket sort itself resolves the fp32 ties.  Either way the tile
    lists must follow the reference order exactly (fp64 depth, then source
    index; rasterizer.py:163, 188-207)."""
    from oracle import fs4d_oracle as O
    rng = np.random.default_rng(11)
    k = 3000
    f32 = lambda a: np.asarray(a, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    if case == "planes":
        depths = rng.choice([3.0, 3.5, 4.0], k)
    else:
        depths = rng.uniform(3.0, 6.0, k)
        depths[rng.choice(k, 40, replace=False)] = 4.0
    cloud = fs().GaussianCloud(
        positions=f32(np.column_stack([rng.uniform(-0.2, 0.2, k), rng.uniform(-0.2, 0.2, k), depths])),
        rotations=f32(q), log_scales=f32(rng.normal(-4.0, 0.3, size=(k, 3))),
        opacity_logits=f32(rng.normal(0.0, 1.0, size=k)), colors_raw=f32(rng.uniform(size=(k, 3))),
        features=f32(rng.normal(size=(k, 4))))
    eps = 1e-7
    T = np.eye(4)
    T[:3, :3] = [[np.cos(eps), 0, np.sin(eps)], [0, 1, 0], [-np.sin(eps), 0, np.cos(eps)]]
    h = w = 64
    fr = frame(h=h, w=w, focal=200.0, T=T)
    out = fs().render(cloud, fr, fs().RasterConfig())
    ocfg = O.RasterParams()
    oproj = O.project(cloud, fr.K, T, h, w, ocfg)
    z32 = oproj["view_depth"].astype(np.float32)
    assert len(z32) - len(np.unique(z32)) > (1000 if case == "planes" else 30)  # the fp32 keys really collide
    olists = O.bin_tiles(oproj, h, w, 16)
    gproj = out.record.proj
    glists = out.record.tile_lists()
    longest = 0
    for ty, row in enumerate(olists):
        for tx, cell in enumerate(row):
            osrc = oproj["source_index"][cell]
            gsrc = gproj.source_index[glists[ty][tx]]
            assert np.array_equal(gsrc, osrc), (ty, tx)
            longest = max(longest, cell.size)
    assert longest > 1000
