#!/bin/bash
# Debug timeline of the tcgen05 MLP (CTA 0, both slots of the two-slot kernel):
# builds a traced libfs4d.so in place on the GPU box, runs one configs[1]
# deform, prints events (who: S<slot> MMA / EPI).
cd "$(dirname "$0")/.."
nvcc -DFS4D_MLP_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared \
  -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
python - <<'PY'
import ctypes, numpy as np, torch, sys
sys.path.insert(0, ".")
import bench
from paper_2503_06161_b200 import device as dv, _native as N
cloud, field, net, K = bench.make_scene(0)
c, f, n = dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net)
eng = dv.DeformEngine()
for _ in range(3):
    eng.forward(c, f, n, 0.3)
lib = N.load()
buf = (ctypes.c_longlong * 2048)(); cnt = (ctypes.c_int * 4)()
lib.fs4d_debug_mlp_trace(buf, cnt)   # reset
eng.forward(c, f, n, 0.3); torch.cuda.synchronize()
lib.fs4d_debug_mlp_trace(buf, cnt)
names = {1: "op-ready", 2: "commit", 3: "acc-ready", 4: "signal"}
ev = []
for who in range(4):
    for i in range(min(cnt[who], 512)):
        v = buf[who * 512 + i]
        ev.append((v >> 4, who, names[v & 15]))
ev.sort()
t0 = ev[0][0]
for t, who, nm in ev[:400]:
    print(f"{t - t0:8d} S{who // 2} {'MMA' if who % 2 == 0 else 'EPI'} {nm}")
print("events", list(cnt), "span", ev[-1][0] - t0)
PY
