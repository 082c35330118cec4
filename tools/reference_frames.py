"""Whole-frame timings of the UNMODIFIED reference CPU path (featsplat 0.1.0,
pip-installed into baseline/_ref) on this host -- SURVEY §8(d) "Reference CPU
path timed beside it":

  * configs[0]: 20 frames (10k Gaussians, 160x128, fx=fy=150, D=8, SH0,
    zero-initialised HexPlane deformation -> identity), t = 0;
  * configs[1]: 3 frames (bench.make_scene: 200k Gaussians, 640x512,
    fx=fy=560, D=16; the reference renders SH degree 0), t = k/155;

each in two modes: one process (NumPy elementwise single-threaded, OpenBLAS
with its default thread count) and P processes over disjoint frames (one
BLAS thread each, P = min(affinity cores, MemAvailable / per-frame RSS,
frames)), as aggregate frames/s.  One frame = deformation.deform +
rasterizer.render (cli.py:58-61).

    python tools/reference_frames.py [--out profiles/r2_reference_frames.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def config0_scene(seed=0):
    """configs[0] as the reference's objects."""
    import featsplat.deformation as RD
    import featsplat.gaussians as RG
    import featsplat.hexplane as RH
    import featsplat.rasterizer as RR
    rng = np.random.default_rng(seed)
    k, h, w, f, d = 10_000, 128, 160, 150.0, 8
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    p = 1.0 / (1.0 + np.exp(-rng.normal(size=k)))
    f32 = bench.f32
    cloud = RG.GaussianCloud(
        positions=f32(np.column_stack([rng.uniform(-1, 1, k), rng.uniform(-1, 1, k), rng.uniform(2, 4, k)])),
        rotations=f32(q), log_scales=f32(rng.normal(-4.0, 0.5, size=(k, 3))),
        opacity_logits=f32(np.log(p) - np.log1p(-p)), colors_raw=f32(rng.uniform(0, 1, size=(k, 3))),
        features=f32(rng.normal(size=(k, d))))
    aabb = np.stack([cloud.positions.min(0), cloud.positions.max(0)])
    aabb = aabb + np.array([[-0.05], [0.05]]) * (aabb[1] - aabb[0])
    field = RH.HexPlaneField(RH.HexPlaneConfig(levels=(1, 2), base_resolution=(64, 64, 64, 25), out_dim=64), aabb, rng)
    field.planes = [[np.zeros_like(pl) for pl in lv] for lv in field.planes]
    net = RD.DeformationNet(64, RD.DeformationConfig(width=64, depth=1, feature_dim=d), rng)
    for _, st in net.stacks():
        for layer in st:
            bound = np.sqrt(6.0 / (layer.in_dim + layer.out_dim))
            layer.weight = f32(rng.uniform(-bound, bound, size=layer.weight.shape))
            layer.bias = np.zeros_like(layer.bias)
    K = np.array([[f, 0, (w - 1) / 2], [0, f, (h - 1) / 2], [0, 0, 1.0]])
    frame = RG.CameraFrame(K=K, T=np.eye(4), time=0.0, image=np.zeros((h, w, 3)), depth=np.zeros((h, w)),
                           mask=np.ones((h, w), dtype=bool))
    return cloud, field, net, frame, RR.RasterConfig()


STATE = {}


def _frame(t):
    import featsplat.deformation as RD
    import featsplat.rasterizer as RR
    import resource
    cloud, field, net, frame, cfg = STATE["scene"]
    t0 = time.perf_counter()
    RR.render(RD.deform(cloud, field, net, float(t)), frame, cfg)
    return time.perf_counter() - t0, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20


def _init_one_thread():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def run(name, scene, ts, frame_gb):
    import multiprocessing as mp
    from threadpoolctl import threadpool_info
    STATE["scene"] = scene
    info = bench.host_info()
    blas = [{k: v for k, v in d.items() if k in ("internal_api", "num_threads", "version")} for d in threadpool_info()]
    # single process, default BLAS threads
    per = [_frame(t) for t in ts]
    single = {"frames": len(ts), "frame_s": [round(x, 3) for x, _ in per], "frames_per_s": len(ts) / sum(x for x, _ in per),
              "peak_rss_gb": round(max(r for _, r in per), 2), "blas": blas}
    procs = max(1, min(info["affinity"], int(info["mem_available_gb"] // frame_gb), len(ts)))
    with mp.get_context("fork").Pool(procs, initializer=_init_one_thread) as pool:
        t0 = time.perf_counter()
        res = pool.map(_frame, list(ts), chunksize=1)
        wall = time.perf_counter() - t0
    multi = {"frames": len(ts), "processes": procs, "blas_threads_per_process": 1, "wall_s": round(wall, 3),
             "frame_s": [round(x, 3) for x, _ in res], "frames_per_s": len(ts) / wall,
             "peak_rss_gb": round(max(r for _, r in res), 2)}
    return {"config": name, "host": info, "single_process": single, "multi_process": multi}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_reference_frames.json"))
    ap.add_argument("--frames0", type=int, default=20)
    ap.add_argument("--frames1", type=int, default=3)
    args = ap.parse_args()
    fsp = bench.load_featsplat()
    if fsp is None:
        raise SystemExit("baseline/_ref (featsplat) not installed")
    out = {"reference": "featsplat 0.1.0 from baseline/_ref, unmodified", "path": "deformation.deform + rasterizer.render"}
    out["configs[0]"] = run("configs[0]", config0_scene(), np.zeros(args.frames0), 2.0)
    out["configs[1]"] = run("configs[1]", bench.reference_scene(0), np.arange(args.frames1) / 155.0,
                            bench.REF_FRAME_GB)
    txt = json.dumps(out, indent=1)
    print(txt)
    with open(args.out, "w") as fh:
        fh.write(txt + "\n")


if __name__ == "__main__":
    main()
