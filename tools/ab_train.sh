#!/bin/bash
# A/B of compile-time knobs on the training step: parity tests on the default
# build, then for each extra-define set a rebuild + the configs[4] train bench.
# usage: bash tools/ab_train.sh "" "-DFS4D_BWD_MINB=8"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_render_parity.py tests/test_gpu_train.py tests/test_gpu_determinism.py tests/test_gpu_headline_parity.py -q -x --timeout 900 2>&1 | tail -2
for defs in "$@"; do
  FS4D_EXTRA_NVCC="$defs" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  for r in 1 2; do
    timeout 300 python bench.py --workload train --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_t.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_t.json').read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print('[$defs]', round(d['value'],2), 'blend_bwd', s.get('blend_bwd'), 'blend', s.get('blend'))"
  done
done
