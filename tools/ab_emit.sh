#!/bin/bash
# A/B of the pair-emission CTA size (rebuilds libfs4d in place on the box).
cd "$(dirname "$0")/.."
for t in 256 512 1024; do
  nvcc -DFS4D_EMIT_THREADS=$t -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
  [ $t = 1024 ] && timeout 600 python -m pytest tests/test_gpu_render_parity.py -q -x 2>&1 | tail -1
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_emit_$t.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_emit_$t.json').read().strip().splitlines()[-1]);print('threads=$t', round(d['value'],1), d['stage_ms']['binning'])"
done
