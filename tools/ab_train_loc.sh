#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_deform_parity.py tests/test_gpu_train.py -q -x --timeout 600 2>&1 | tail -3
for v in 1 0; do
  FS4D_TRAIN_LOCALITY=$v timeout 300 python bench.py --workload train --steps 5 --warmup 3 --no-cpu > gpurun_out/ab_tl_$v.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_tl_$v.json').read().strip().splitlines()[-1]);print('locality=$v', round(d['value'],2), d['stage_ms_per_step'])"
done
