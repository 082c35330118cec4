"""GPU parity of adaptive density control (gaussians.py:309-425 on device,
csrc/density.cu) against the reference's goldens and the float64 oracle:
classification decisions and the output row order are exact; split-child
positions / log-scales are fp32 roundings of the fp64 values (1e-6 relative);
everything copied is bit-exact."""

import numpy as np
import pytest

from conftest import CLOUD_FIELDS, has_gpu, load_golden, random_cloud_arrays
from oracle import fs4d_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def _close(a, b, rel=1e-6, what=""):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    err = np.abs(a - b).max() if a.size else 0.0
    assert err <= rel * max(1.0, np.abs(b).max() if b.size else 1.0), (what, err)


def test_densify_and_prune_matches_reference_goldens():
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import density as dn
    from paper_2503_06161_b200.numerics import AdamState
    g = load_golden("density")
    cloud = fs.GaussianCloud(**{f: g[f"cloud_{f}"].copy() for f in CLOUD_FIELDS})
    stats = dn.ViewspaceGradStats(g["stats_accum"].copy(), g["stats_count"].copy())
    adam = {f: AdamState(m=g[f"adam_{f}_m"].copy(), v=g[f"adam_{f}_v"].copy()) for f in CLOUD_FIELDS}
    thr, pd, po, sf, ext = g["cfg"]
    cfg = dn.DensityControlConfig(thr, pd, po, sf)
    rep = dn.densify_and_prune(cloud, stats, 5, cfg, ext, np.random.default_rng(int(g["split_seed"])),
                               adam_states=adam)
    assert [rep["cloned"], rep["split"], rep["pruned"], rep["count"]] == list(g["report"])
    for f in CLOUD_FIELDS:
        if f in ("positions", "log_scales"):
            _close(getattr(cloud, f), g[f"out_{f}"], 1e-6, f)
        else:
            np.testing.assert_array_equal(getattr(cloud, f), g[f"out_{f}"], err_msg=f)
        np.testing.assert_array_equal(adam[f].m, g[f"out_adam_{f}_m"])
        np.testing.assert_array_equal(adam[f].v, g[f"out_adam_{f}_v"])
    assert len(stats.accum) == rep["count"] and not stats.accum.any() and not stats.count.any()


def test_prune_only_and_reset_opacity_match_reference_goldens():
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import density as dn
    g = load_golden("density")
    arrs = {f: g[f"out_{f}"].astype(np.float32).astype(np.float64) for f in CLOUD_FIELDS}
    arrs["opacity_logits"] = g["po_in_opacity"].copy()
    cloud = fs.GaussianCloud(**arrs)
    stats = dn.ViewspaceGradStats(g["po_accum"].copy(), g["po_count"].copy())
    n = dn.prune_only(cloud, stats, dn.DensityControlConfig(prune_opacity=float(g["cfg"][2])))
    assert n == int(g["po_pruned"])
    np.testing.assert_array_equal(stats.accum, g["po_out_accum"])
    np.testing.assert_array_equal(stats.count, g["po_out_count"])
    _close(cloud.positions, g["po_out_positions"], 1e-7, "positions")
    cloud.opacity_logits = g["ro_in"].copy()
    dn.reset_opacity(cloud, 0.01)
    _close(cloud.opacity_logits, g["ro_out"], 1e-6, "reset_opacity")


def test_device_density_full_size_matches_oracle():
    """200k Gaussians with SH3 rows and two extra per-row arrays."""
    import torch
    from paper_2503_06161_b200 import density as dn
    from paper_2503_06161_b200.device import DeviceCloud
    rng = np.random.default_rng(9)
    k = 200_000
    a = random_cloud_arrays(rng, k, 16, op_range=(0.001, 0.9), ls_range=(0.002, 0.2), sh_degree=3)
    import paper_2503_06161_b200 as fs
    cloud = DeviceCloud.from_cloud(fs.GaussianCloud(**a))
    acc = rng.exponential(3e-4, size=k)
    cnt = np.floor(rng.uniform(0, 4, size=k))
    stats = dn.ViewspaceGradStats(torch.tensor(acc, device="cuda"), torch.tensor(cnt, device="cuda"))
    ex = [rng.normal(size=(k, 3)).astype(np.float32), rng.normal(size=(k,)).astype(np.float32)]
    cfg = dn.DensityControlConfig(2e-4, 0.05, 0.02, 1.6)
    out, st, outs, rep = dn.DeviceDensity().run(cloud, stats, cfg, 1.3, np.random.default_rng(5), False,
                                                 [torch.tensor(e, device="cuda") for e in ex])
    zrng = np.random.default_rng(5)
    ref_cloud = fs.GaussianCloud(**a)
    ro, racc, rcnt, rex, rc = O.density_control(ref_cloud, acc, cnt, 2e-4, 0.05, 0.02, 1.6, 1.3,
                                                np.stack([zrng.standard_normal((rep["split"], 3)) for _ in range(2)]),
                                                extras=[e.astype(np.float64) for e in ex])
    assert (rep["cloned"], rep["split"], rep["count"]) == (rc["clone"], rc["split"], len(ro["positions"]))
    assert rep["pruned"] == rc["pruned"]
    for f in CLOUD_FIELDS + ("sh_rest",):
        got = getattr(out, f).cpu().numpy().astype(np.float64)
        if f in ("positions", "log_scales"):
            _close(got, ro[f], 1e-6, f)
        else:
            np.testing.assert_array_equal(got.reshape(ro[f].shape), ro[f], err_msg=f)
    for o, r in zip(outs, rex):
        np.testing.assert_array_equal(o.cpu().numpy().astype(np.float64), r)
    assert not st.accum.any() and not st.count.any()


def test_grad_stats_add_device_matches_numpy():
    import torch
    from paper_2503_06161_b200 import density as dn
    rng = np.random.default_rng(2)
    k = 50_000
    host = dn.ViewspaceGradStats.zeros(k)
    dev = dn.ViewspaceGradStats.zeros(k, "cuda")
    for _ in range(4):
        idx = rng.permutation(k)[:20_000].astype(np.int32)
        nrm = rng.uniform(size=20_000).astype(np.float32)
        host.add(idx, nrm.astype(np.float64))
        dev.add(torch.tensor(idx, device="cuda"), torch.tensor(nrm, device="cuda"))
    np.testing.assert_array_equal(dev.accum.cpu().numpy(), host.accum)
    np.testing.assert_array_equal(dev.count.cpu().numpy(), host.count)
