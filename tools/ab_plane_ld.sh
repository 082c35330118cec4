#!/bin/bash
cd "$(dirname "$0")/.."
for m in __ldg __ldcg __ldlu; do
  nvcc "-DPLANE_LD=$m" -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
  timeout 300 python bench.py --no-cpu > gpurun_out/ab_pl_$m.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_pl_$m.json').read().strip().splitlines()[-1]);print('$m', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms']['deform_gather'])"
done
