"""Pin the oracle's density-control restatement (gaussians.py:349-425) to the
reference's own outputs (tests/golden/make_golden.py density_case).  CPU only."""

from types import SimpleNamespace

import numpy as np

from conftest import CLOUD_FIELDS, load_golden
from oracle import fs4d_oracle as O


def _normals(g):
    rng = np.random.default_rng(int(g["split_seed"]))
    n = int(g["report"][1])
    return np.stack([rng.standard_normal((n, 3)) for _ in range(2)])


def test_oracle_densify_matches_reference():
    g = load_golden("density")
    cloud = SimpleNamespace(**{f: g[f"cloud_{f}"] for f in CLOUD_FIELDS}, sh_rest=None)
    thr, pd, po, sf, ext = g["cfg"]
    extras = [g[f"adam_{f}_{t}"] for f in CLOUD_FIELDS for t in ("m", "v")]
    out, acc, cnt, ex, counts = O.density_control(cloud, g["stats_accum"], g["stats_count"], thr, pd, po, sf, ext,
                                                  _normals(g), extras=extras)
    assert [counts["clone"], counts["split"], counts["pruned"], len(out["positions"])] == list(g["report"])
    for f in CLOUD_FIELDS:
        np.testing.assert_allclose(out[f], g[f"out_{f}"], rtol=0, atol=1e-14, err_msg=f)
    i = 0
    for f in CLOUD_FIELDS:
        for t in ("m", "v"):
            np.testing.assert_array_equal(ex[i], g[f"out_adam_{f}_{t}"])
            i += 1
    assert not acc.any() and not cnt.any() and len(acc) == len(g["out_accum"])


def test_oracle_prune_only_matches_reference():
    g = load_golden("density")
    cloud = SimpleNamespace(**{f: g[f"out_{f}"] for f in CLOUD_FIELDS}, sh_rest=None)
    cloud.opacity_logits = g["po_in_opacity"]
    po = g["cfg"][2]
    out, acc, cnt, _, counts = O.density_control(cloud, g["po_accum"], g["po_count"], 0, 0, po, 1.6, 1.0,
                                                 prune_only=True)
    assert len(g["po_in_opacity"]) - counts["keep"] == int(g["po_pruned"])
    np.testing.assert_array_equal(acc, g["po_out_accum"])
    np.testing.assert_array_equal(cnt, g["po_out_count"])
    np.testing.assert_array_equal(out["positions"], g["po_out_positions"])


def test_host_density_config_defaults():
    from paper_2503_06161_b200.density import DensityControlConfig
    c = DensityControlConfig()
    assert (c.grad_threshold, c.percent_dense, c.prune_opacity, c.split_factor) == (2e-4, 0.01, 0.005, 1.6)
