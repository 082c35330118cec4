import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

CLOUD_FIELDS = ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfs4d.so")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_cloud(g):
    return SimpleNamespace(**{f: g[f"cloud_{f}"] for f in CLOUD_FIELDS}, sh_rest=None)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def random_cloud_arrays(rng, k, nf, op_range=(0.05, 0.98), depth_range=(2.2, 3.8), xy=0.9,
                        ls_range=(0.08, 0.35), sh_degree=0, sh_sigma=0.2):
    pos = np.column_stack([rng.uniform(-xy, xy, k), rng.uniform(-xy, xy, k),
                           rng.uniform(*depth_range, k)])
    p = rng.uniform(*op_range, k)
    d = dict(positions=f32(pos), rotations=f32(rng.normal(size=(k, 4))),
             log_scales=f32(np.log(rng.uniform(*ls_range, size=(k, 3)))),
             opacity_logits=f32(np.log(p) - np.log1p(-p)),
             colors_raw=f32(rng.uniform(0.1, 0.9, size=(k, 3))),
             features=f32(rng.normal(size=(k, nf))))
    n_sh = (sh_degree + 1) ** 2 - 1
    d["sh_rest"] = f32(rng.normal(size=(k, n_sh, 3)) * sh_sigma) if n_sh else None
    return d


def pinhole(h, w, focal):
    return np.array([[focal, 0, (w - 1) / 2], [0, focal, (h - 1) / 2], [0, 0, 1.0]])


def rigid_T(rng, max_deg=5.0, max_t=0.1):
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = np.deg2rad(rng.uniform(-max_deg, max_deg))
    Kx = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + np.sin(ang) * Kx + (1 - np.cos(ang)) * Kx @ Kx
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = rng.uniform(-max_t, max_t, 3)
    return T


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
