#!/bin/bash
# Phase timeline (clock64) of the densest tile's sort CTA (and its bucket
# statistics): builds a traced libfs4d.so in place on the GPU box, renders
# the configs[1] scene, prints cycles from CTA entry per phase.
cd "$(dirname "$0")/.."
nvcc -DFS4D_SORT_TRACE $FS4D_EXTRA_NVCC -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  -shared -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
python - <<'PY'
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np, bench
import paper_2503_06161_b200 as fs
from paper_2503_06161_b200 import _native as N
cloud, field, net, K = bench.make_scene(0)
H, W = bench.H, bench.W
cam = fs.CameraFrame(K=K, T=np.eye(4), time=0.0, image=np.zeros((H, W, 3)), depth=np.zeros((H, W)),
                     mask=np.ones((H, W), bool))
for _ in range(3):
    out = fs.render(cloud, cam, fs.RasterConfig())
lib = N.load()
buf = (ctypes.c_longlong * 32)()
lib.fs4d_debug_sort_trace(buf)
for o, name in ((0, "densest tile"), (16, "CTA FS4D_SORT_TRACE2")):
    t = [buf[o + i] for i in range(16)]
    print(name, "phase cycles from entry:", [t[i] - t[0] if t[i] else None for i in range(12)])
    print(name, "bmax, NB, n, kmax-kmin:", t[12:16])
PY
