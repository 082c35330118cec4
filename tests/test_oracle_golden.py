"""Pin the CPU oracle (oracle/fs4d_oracle.py) to golden vectors produced by
the reference implementation itself (tests/golden/make_golden.py).  CPU only."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cloud, load_golden
from oracle import fs4d_oracle as O

RENDER_CASES = sorted(os.path.basename(p)[len("render_"):-4]
                      for p in glob.glob(os.path.join(GOLDEN, "render_*.npz")))
DEFORM_CASES = sorted(os.path.basename(p)[len("deform_"):-4]
                      for p in glob.glob(os.path.join(GOLDEN, "deform_*.npz")))


def test_fixtures_present():
    assert len(RENDER_CASES) >= 6 and len(DEFORM_CASES) >= 2


@pytest.mark.parametrize("case", RENDER_CASES)
def test_oracle_render_matches_reference(case):
    g = load_golden("render_" + case)
    cfg = O.RasterParams(background=g["background"])
    cloud = golden_cloud(g)
    h, w = int(g["height"]), int(g["width"])
    out = O.render(cloud, g["K"], g["T"], h, w, cfg)
    proj = out["proj"]
    np.testing.assert_array_equal(proj["source_index"], g["proj_source_index"])
    np.testing.assert_array_equal(proj["radius"], g["proj_radius"])
    np.testing.assert_allclose(proj["mean2d"], g["proj_mean2d"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(proj["conic"], g["proj_conic"], rtol=1e-10, atol=1e-12)
    lists = O.bin_tiles(proj, h, w, 16)
    flat = [cell for row in lists for cell in row]
    rows = np.concatenate(flat) if flat else np.zeros(0, np.int64)
    np.testing.assert_array_equal(rows, g["tile_rows"])
    np.testing.assert_array_equal([c.size for c in flat], g["tile_ranges"][:, 1] - g["tile_ranges"][:, 0])
    for key in ("color", "depth", "feature", "alpha"):
        np.testing.assert_allclose(out[key], g[key], rtol=0, atol=1e-10, err_msg=key)
    np.testing.assert_array_equal(out["n_contrib"], g["n_contrib"])
    if "grad_positions" in g:
        gr = O.render_backward(cloud, g["K"], g["T"], h, w, cfg, out, g["up_color"], g["up_depth"],
                               g["up_feature"], g["up_alpha"])
        for f in ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features",
                  "viewspace_norm"):
            ref = g[f"grad_{f}"]
            scale = max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(gr[f], ref, rtol=0, atol=1e-9 * scale, err_msg=f)
        np.testing.assert_array_equal(gr["viewspace_index"], g["grad_viewspace_index"])


def _golden_net(g):
    net = {}
    for key in g:
        if key.startswith("w:"):
            prefix, i = key[2:].rsplit(".", 1)
            net.setdefault(prefix, {})[int(i)] = key
    out = {}
    for prefix, layers in net.items():
        stack = []
        for i in sorted(layers):
            relu = not (prefix.startswith("net.head") or (prefix == "net.feat" and i == 1))
            stack.append((g[f"w:{prefix}.{i}"], g[f"b:{prefix}.{i}"], relu))
        out[prefix] = stack
    return out


def _golden_planes(g):
    levels = len(g["levels"])
    return [[g[f"plane_{l}_{p}"] for p in range(6)] for l in range(levels)]


@pytest.mark.parametrize("case", DEFORM_CASES)
def test_oracle_deform_matches_reference(case):
    g = load_golden("deform_" + case)
    cloud = golden_cloud(g)
    planes, net = _golden_planes(g), _golden_net(g)
    t = float(g["t"])
    lat = O.hexplane_query(planes, g["aabb"], cloud.positions, t)
    np.testing.assert_allclose(lat, g["latent"], rtol=1e-12, atol=1e-14)
    snap, cache = O.deform(cloud, planes, g["aabb"], net, t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        np.testing.assert_allclose(snap[f], g[f"snap_{f}"], rtol=1e-12, atol=1e-12, err_msg=f)
    ups = {f: g[f"up_{f}"] for f in ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    cg, ng, pg = O.deform_backward(cloud, planes, g["aabb"], net, cache, ups)
    np.testing.assert_allclose(cg["positions"], g["cg_positions"], rtol=1e-10, atol=1e-10)
    for key in g:
        if key.startswith("g:"):
            np.testing.assert_allclose(ng[key[2:]], g[key], rtol=1e-10, atol=1e-10, err_msg=key)
    for l, level in enumerate(pg):
        for p, arr in enumerate(level):
            np.testing.assert_allclose(arr, g[f"gplane_{l}_{p}"], rtol=1e-10, atol=1e-10)


def test_oracle_sh_degree0_reduces_to_reference_colour():
    g = load_golden("render_s1")
    cloud = golden_cloud(g)
    cloud.sh_rest = np.zeros((cloud.positions.shape[0], 15, 3))
    cfg = O.RasterParams(background=g["background"])
    out = O.render(cloud, g["K"], g["T"], int(g["height"]), int(g["width"]), cfg)
    np.testing.assert_allclose(out["color"], g["color"], atol=1e-12)


HEX_EDGE_CASES = ["t0", "t1", "tclip"]


@pytest.mark.parametrize("case", HEX_EDGE_CASES)
def test_oracle_hexplane_edges_match_reference(case):
    """Outside-aabb / on-face Gaussians and t at (and past) the ends of [0, 1]
    (hexplane.py:84-110, 145-187; make_golden.hexplane_edge_case)."""
    g = load_golden("hexplane_" + case)
    cloud = golden_cloud(g)
    planes, net = _golden_planes(g), _golden_net(g)
    t = float(g["t"])
    coords, inside = O.field_coords(g["aabb"], cloud.positions, t)
    np.testing.assert_array_equal(coords, g["coords"])
    np.testing.assert_array_equal(inside, g["inside"])
    assert (~inside).any(axis=1).sum() >= 20
    lat = O.hexplane_query(planes, g["aabb"], cloud.positions, t)
    np.testing.assert_allclose(lat, g["latent"], rtol=1e-12, atol=1e-14)
    pg, dpos = O.hexplane_backward(planes, g["aabb"], cloud.positions, t, g["d_latent"])
    np.testing.assert_allclose(dpos, g["query_dpos"], rtol=1e-10, atol=1e-12)
    assert np.all(dpos[~inside] == 0.0)  # clamped coordinates pass no position gradient
    for l, level in enumerate(pg):
        for p, arr in enumerate(level):
            np.testing.assert_allclose(arr, g[f"qgplane_{l}_{p}"], rtol=1e-10, atol=1e-12)
    snap, cache = O.deform(cloud, planes, g["aabb"], net, t)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
        np.testing.assert_allclose(snap[f], g[f"snap_{f}"], rtol=1e-12, atol=1e-12, err_msg=f)
    ups = {f: g[f"up_{f}"] for f in ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    cg, ng, pg = O.deform_backward(cloud, planes, g["aabb"], net, cache, ups)
    np.testing.assert_allclose(cg["positions"], g["cg_positions"], rtol=1e-10, atol=1e-10)
    for key in g:
        if key.startswith("g:"):
            np.testing.assert_allclose(ng[key[2:]], g[key], rtol=1e-10, atol=1e-10, err_msg=key)
    for l, level in enumerate(pg):
        for p, arr in enumerate(level):
            np.testing.assert_allclose(arr, g[f"gplane_{l}_{p}"], rtol=1e-10, atol=1e-10)
