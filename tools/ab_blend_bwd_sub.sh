#!/bin/bash
# A/B of CTAs per tile in the blend backward (FS4D_BLEND_BWD_SUB).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FS4D_BLEND_BWD_SUB=4 timeout 600 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_train.py -q -x 2>&1 | tail -1
for sb in 1 2 4; do
  FS4D_BLEND_BWD_SUB=$sb timeout 300 python bench.py --workload train --no-cpu > gpurun_out/ab_bsub_$sb.json 2>&1
  FS4D_BLEND_BWD_SUB=$sb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_blend_bwd2" -s 4 -c 4 --csv --log-file gpurun_out/ab_bsub_$sb.csv python bench.py --workload train --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
  echo "sub=$sb $(python -c "import json;d=json.loads(open('gpurun_out/ab_bsub_$sb.json').read().strip().splitlines()[-1]);print(round(d['value'],2), d['stage_ms_per_step']['blend_bwd'])") $(python tools/ncu_summary.py launches gpurun_out/ab_bsub_$sb.csv | tail -1)"
done
