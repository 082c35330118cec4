#!/bin/bash
# Preprocess occupancy A/B (FS4D_PRE_MINB) + frames-in-flight A/B (FS4D_SEQ_STREAMS) on the render bench.
mkdir -p gpurun_out
bash tools/ab_define.sh "-DFS4D_PRE_MINB=4" ""
timeout 1200 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_headline_parity.py tests/test_gpu_edge_cases.py -q -x --timeout 900 2>&1 | tail -2
for n in 2 4; do
  FS4D_SEQ_STREAMS=$n timeout 300 python bench.py --no-cpu > gpurun_out/ab_s.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_s.json').read().strip().splitlines()[-1]);print('streams=$n', round(d['value'],1))"
done
