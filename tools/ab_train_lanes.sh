#!/bin/bash
# A/B of training pairs in flight (FS4D_TRAIN_LANES): steps/s for configs[4] and the fine stage.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_density.py -q -x 2>&1 | tail -2
for l in 1 2 3; do
  for wl in train fine; do
    FS4D_TRAIN_LANES=$l timeout 300 python bench.py --workload $wl --no-cpu > gpurun_out/ab_lanes_${wl}_$l.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_lanes_${wl}_$l.json').read().strip().splitlines()[-1]);print('$wl lanes=$l', round(d['value'],2))"
  done
done
