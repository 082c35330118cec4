#!/bin/bash
# Host-side enqueue cost per frame of the resident pipeline (is the CPU the limit?).
python - <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench
import paper_2503_06161_b200 as fs
from paper_2503_06161_b200 import device as dv
cloud_np, field_np, net_np, K = bench.make_scene(0)
c, f, n = dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np), dv.DeviceNet.from_net(net_np)
seq = dv.SequenceRenderer(c, f, n, 512, 640, fs.RasterConfig(), pipelines=6, streams=3, replicas=6)
seq.warm(0.1, K, np.eye(4))
ts = [i / 155 for i in range(120)]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = seq.run(ts, K, np.eye(4))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e6*(t1-t0)/len(ts):.1f} us/frame, wall {1e6*(t2-t0)/len(ts):.1f} us/frame, gpu {1e3*a.elapsed_time(b)/len(ts):.1f} us/frame")
PY
