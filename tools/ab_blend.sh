#!/bin/bash
# A/B of blend variants (FS4D_BLEND_SUB) with the parity tests first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_edge_cases.py -q -x --timeout 600 2>&1 | tail -4
for sub in 2 4 1; do
  FS4D_BLEND_SUB=$sub timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_blend_$sub.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_blend_$sub.json'));print('sub=$sub', round(d['value'],1), d['stage_ms'])"
done
