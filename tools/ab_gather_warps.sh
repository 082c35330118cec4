#!/bin/bash
# A/B of the HexPlane gather CTA size (rebuilds libfs4d in place on the box).
cd "$(dirname "$0")/.."
for w in 4 2 8; do
  nvcc -DFS4D_GATHER_WARPS=$w -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_gw_$w.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_gw_$w.json').read().strip().splitlines()[-1]);print('warps=$w', round(d['value'],1), d['stage_ms']['deform_gather'])"
done
