#!/bin/bash
# Frames in flight: 1 stream vs 2 streams (independent frame pipelines), with 3
# rotating model replicas (3 x 70 MB > L2) so no L2 flush is needed either way.
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
import paper_2503_06161_b200 as fs
from paper_2503_06161_b200 import device as dv
cloud_np, field_np, net_np, K = bench.make_scene(0)
reps = []
for r in range(3):
    reps.append((dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np), dv.DeviceNet.from_net(net_np)))
cfg = fs.RasterConfig()
T = np.eye(4)
reps.append((dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np), dv.DeviceNet.from_net(net_np)))
reps += [(dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np), dv.DeviceNet.from_net(net_np)) for _ in range(2)]
pipes = [dv.FramePipeline(*reps[r], 512, 640, cfg) for r in range(6)]
for p in pipes:
    p.run(0.1, K, T, check=True)
    p.renderer.cap = p.renderer.cap
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in range(3)]
def run(nstreams, n=60):
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(cur)
    for s in streams: s.wait_event(a)
    for i in range(n):
        p = i % 6
        with torch.cuda.stream(streams[p % nstreams]):
            pipes[p].run(i / 59.0, K, T)
    for s in streams: cur.wait_stream(s)
    b.record(cur)
    torch.cuda.synchronize()
    return n / (a.elapsed_time(b) / 1000.0)
for rep in range(1):
    print("1 stream  frames/s", round(run(1), 1))
    print("2 streams frames/s", round(run(2), 1))
    print("3 streams frames/s", round(run(3), 1))
PY
