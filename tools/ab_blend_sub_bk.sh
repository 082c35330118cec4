#!/bin/bash
# A/B of CTAs per tile in the blend forward (FS4D_BLEND_SUB) at the current
# group size, each setting twice.
mkdir -p gpurun_out
for sb in 2 1 4 2 1 4; do
  FS4D_BLEND_SUB=$sb timeout 300 python bench.py --no-cpu > gpurun_out/ab_sub.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_sub.json').read().strip().splitlines()[-1]);print('sub=$sb', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms']['blend'])"
done
