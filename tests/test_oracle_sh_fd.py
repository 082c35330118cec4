"""Finite-difference pin of the SH extension: the
reference has no SH, so the oracle's degree 1-3 colour term and
its gradients -- which the device is compared against -- are checked here
against central differences of the oracle's own float64 render.  Gradients
w.r.t. the SH coefficients and, through the view direction, the positions.
CPU only."""

import numpy as np
import pytest

from conftest import pinhole, random_cloud_arrays
from oracle import fs4d_oracle as O


def _loss(arrs, K, T, h, w, cfg, up):
    out = O.render(type("C", (), arrs)(), K, T, h, w, cfg)
    return float(np.sum(up * out["color"]))


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_sh_gradients_match_central_differences(degree):
    rng = np.random.default_rng(40 + degree)
    h, w = 24, 28
    arrs = random_cloud_arrays(rng, 6, 3, op_range=(0.2, 0.6), depth_range=(2.5, 3.5), xy=0.4,
                               ls_range=(0.15, 0.3), sh_degree=degree, sh_sigma=0.15)
    # keep the raw colours well inside (0, 1): the clamp gate is then open for
    # every Gaussian and the loss is smooth in the SH coefficients
    arrs["colors_raw"] = np.full_like(arrs["colors_raw"], 0.5)
    K = pinhole(h, w, 30.0)
    T = np.eye(4)
    T[:3, 3] = [0.05, -0.03, 0.1]
    cfg = O.RasterParams()
    up = rng.normal(size=(h, w, 3))
    out = O.render(type("C", (), arrs)(), K, T, h, w, cfg)
    g = O.render_backward(type("C", (), arrs)(), K, T, h, w, cfg, out, up)
    eps = 1e-6
    sh = arrs["sh_rest"]
    flat = sh.reshape(-1)
    fd = np.empty(flat.size)
    for i in range(flat.size):
        old = flat[i]
        flat[i] = old + eps
        fp = _loss(arrs, K, T, h, w, cfg, up)
        flat[i] = old - eps
        fm = _loss(arrs, K, T, h, w, cfg, up)
        flat[i] = old
        fd[i] = (fp - fm) / (2 * eps)
    ga = g["sh_rest"].reshape(-1)
    assert np.abs(ga - fd).max() < 1e-6 * max(1.0, np.abs(fd).max()), np.abs(ga - fd).max()
    # positions: the SH term's view-direction dependence adds to the projection chain
    pos = arrs["positions"].reshape(-1)
    fdp = np.empty(pos.size)
    for i in range(pos.size):
        old = pos[i]
        pos[i] = old + eps
        fp = _loss(arrs, K, T, h, w, cfg, up)
        pos[i] = old - eps
        fm = _loss(arrs, K, T, h, w, cfg, up)
        pos[i] = old
        fdp[i] = (fp - fm) / (2 * eps)
    gp = g["positions"].reshape(-1)
    assert np.abs(gp - fdp).max() < 1e-4 * max(1.0, np.abs(fdp).max()), np.abs(gp - fdp).max()
