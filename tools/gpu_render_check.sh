#!/bin/bash
# Render-path GPU check after a forward-kernel change: render / headline / edge
# parity, then the render bench (default and FS4D_SEQ_STREAMS=4).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_headline_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_reference_api.py -q -x --timeout 900 2>&1 | tail -2
for n in 3 4 3 4; do
  FS4D_SEQ_STREAMS=$n timeout 300 python bench.py --no-cpu > gpurun_out/rc.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/rc.json').read().strip().splitlines()[-1]);print('streams=$n', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms'])"
done
