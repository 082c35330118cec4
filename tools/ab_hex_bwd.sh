#!/bin/bash
# A/B of the HexPlane backward: time rows on/off, 1 or 2 resident CTAs per SM.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_deform_parity.py -q -x 2>&1 | tail -2
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --workload train --no-cpu > gpurun_out/ab_hex_$tag.json 2>&1
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hexplane_bwd_c32" -c 6 --csv --log-file gpurun_out/ab_hex_$tag.csv python bench.py --workload train --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
  echo "$tag $(python -c "import json;d=json.loads(open('gpurun_out/ab_hex_$tag.json').read().strip().splitlines()[-1]);print(round(d['value'],2), d['stage_ms_per_step']['deform_bwd'])") $(python tools/ncu_summary.py launches gpurun_out/ab_hex_$tag.csv | tail -1)"
}
run rows
run norows FS4D_NO_TIME_ROWS=1
nvcc -DFS4D_HEX_BWD_MINB=2 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -o paper_2503_06161_b200/libfs4d.so paper_2503_06161_b200/csrc/*.cu || exit 1
run minb2
