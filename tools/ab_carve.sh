#!/bin/bash
# Gather L1/shared carveout A/B (FS4D_GATHER_CARVEOUT percent; unset = driver default).
mkdir -p gpurun_out
for c in -1 25 50 75 -1; do
  if [ $c = -1 ]; then unset FS4D_GATHER_CARVEOUT; else export FS4D_GATHER_CARVEOUT=$c; fi
  timeout 300 python bench.py --no-cpu > gpurun_out/ac.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ac.json').read().strip().splitlines()[-1]);print('carveout=$c', round(d['value'],1), d['stage_ms']['deform_gather'])"
done
