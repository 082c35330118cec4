#!/bin/bash
cd "$(dirname "$0")" 2>/dev/null; cd /root/repo
for bk in 4 8 2; do
  nvcc -DFS4D_BLEND_BK=$bk -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
  [ $bk = 8 ] && timeout 600 python -m pytest tests/test_gpu_render_parity.py -q -x 2>&1 | tail -1
  timeout 300 python bench.py --no-cpu > gpurun_out/ab_bk_$bk.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_bk_$bk.json').read().strip().splitlines()[-1]);print('bk=$bk', round(d['value'],1), round(d['value_serial']['value'],1), d['stage_ms']['blend'])"
done
