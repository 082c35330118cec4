#!/bin/bash
# Launch-bound minimums A/B: blend forward (render bench) and blend backward (train bench).
bash tools/ab_define.sh "-DFS4D_BLEND_MINB=7" "-DFS4D_BLEND_MINB=6" ""
for defs in "-DFS4D_BWD_MINB=9" "-DFS4D_BWD_MINB=10" ""; do
  FS4D_EXTRA_NVCC="$defs" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  timeout 300 python bench.py --workload train --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_t.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_t.json').read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print('[$defs]', round(d['value'],2), 'blend_bwd', s.get('blend_bwd'))"
done
