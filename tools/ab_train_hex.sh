#!/bin/bash
# A/B of the HexPlane-backward knobs on the training step: for each extra-define
# set, rebuild, then train bench with the locality order off / on.
# usage: bash tools/ab_train_hex.sh "" "-DFS4D_HEX_BWD_MINB=1"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_deform_parity.py tests/test_gpu_train.py tests/test_gpu_headline_parity.py -q -x --timeout 600 2>&1 | tail -2
for defs in "$@"; do
  FS4D_EXTRA_NVCC="$defs" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  for v in 0 1; do
    FS4D_TRAIN_LOCALITY=$v timeout 300 python bench.py --workload train --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_th.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_th.json').read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print('[$defs] loc=$v', round(d['value'],2), 'deform_bwd', s.get('deform_bwd'), 'fwd', s.get('deform_fwd'))"
  done
done
