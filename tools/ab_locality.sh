#!/bin/bash
# A/B of the HexPlane gather visiting order (index order vs Morton locality order).
mkdir -p gpurun_out
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2503_06161_b200 import device as dv
cloud, field, net, K = bench.make_scene(0)
c, f, n = dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net)
order = dv.locality_order(c.positions, f.aabb)
o = order.cpu().numpy()
assert np.array_equal(np.sort(o), np.arange(len(o))), "not a permutation"
e = dv.DeformEngine()
a = e.forward(c, f, n, 0.37)
b = e.forward(c, f.with_order(order), n, 0.37)
torch.cuda.synchronize()
for name in ("positions", "rotations", "log_scales", "opacity_logits", "features"):
    assert torch.equal(getattr(a, name), getattr(b, name)), name
print("order is a permutation; deform outputs bit-identical with and without it")
PY
for v in 0 1; do
  FS4D_LOCALITY=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_loc_$v.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_loc_$v.json').read().strip().splitlines()[-1]);print('locality=$v', round(d['value'],1), d['stage_ms'])"
done
