#!/bin/bash
for g in 148 111 74; do
  FS4D_MLP_GRID=$g timeout 300 python bench.py --no-cpu > gpurun_out/ab_mg_$g.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_mg_$g.json').read().strip().splitlines()[-1]);print('grid=$g', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms']['deform_mlp'])"
done
