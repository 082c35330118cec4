#!/bin/bash
# A/B of blend variants: FS4D_BLEND_PX (pixels per thread) x FS4D_BLEND_SUB (CTAs per tile).
mkdir -p gpurun_out
FS4D_BLEND_PX=2 timeout 900 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_edge_cases.py -q -x --timeout 600 2>&1 | tail -3
for cfg in "1 2" "2 1" "2 2" "2 4"; do
  set -- $cfg
  FS4D_BLEND_PX=$1 FS4D_BLEND_SUB=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_blend_$1_$2.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_blend_$1_$2.json').read().strip().splitlines()[-1]);print('px=$1 sub=$2', round(d['value'],1), d['stage_ms']['blend'])"
done
