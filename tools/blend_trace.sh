#!/bin/bash
# Per-CTA timeline of k_blend at configs[1] (debug build in place on the GPU box).
cd "$(dirname "$0")/.."
nvcc -DFS4D_BLEND_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared \
  -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
python - <<'PY'
import ctypes, numpy as np, torch, sys
sys.path.insert(0, ".")
import bench
import paper_2503_06161_b200 as fs
from paper_2503_06161_b200 import device as dv, _native as N
cloud, field, net, K = bench.make_scene(0)
c = dv.DeviceCloud.from_cloud(cloud)
r = dv.Renderer()
for _ in range(3):
    imgs, rec = r.forward(c, K, np.eye(4), 512, 640, fs.RasterConfig(), check=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8192 * 4))()
N.load().fs4d_debug_blend_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 4)[:2560].astype(np.float64)
t0 = a[:, 0].min()
st, en, sm, nb = a[:, 0] - t0, a[:, 1] - t0, a[:, 2], a[:, 3]
dur = en - st
print("kernel span us", en.max() / 1e3, "start spread us", st.max() / 1e3)
print("cta dur us pct 50/90/99/100", np.percentile(dur, [50, 90, 99, 100]) / 1e3)
print("batches pct 50/90/99/100", np.percentile(nb, [50, 90, 99, 100]))
order = np.argsort(-dur)[:10]
for i in order:
    print(f"cta {i} tile {i//2} start {st[i]/1e3:.1f} dur {dur[i]/1e3:.1f} us batches {nb[i]:.0f} sm {sm[i]:.0f}")
# per-SM busy time
busy = np.zeros(148)
for i in range(2560):
    busy[int(sm[i])] = max(busy[int(sm[i])], en[i])
print("SM finish us pct 0/50/100", np.percentile(busy, [0, 50, 100]) / 1e3)
# time at which 90% of CTAs are done
print("90% CTAs done at us", np.percentile(en, 90) / 1e3, "99%", np.percentile(en, 99) / 1e3)
PY
