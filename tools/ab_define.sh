#!/bin/bash
# A/B of compile-time knobs: for each "-DNAME=VALUE ..." argument, rebuild
# libfs4d.so on the box with those extra nvcc defines and print the render
# bench value and stage times.  usage: bash tools/ab_define.sh "" "-DFS4D_BLEND_MINB=8"
mkdir -p gpurun_out
for defs in "$@"; do
  FS4D_EXTRA_NVCC="$defs" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  timeout 300 python bench.py --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('[$defs]', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms'])"
done
