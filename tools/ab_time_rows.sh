#!/bin/bash
# A/B of the HexPlane gather with / without the per-frame time rows.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_deform_parity.py tests/test_gpu_train.py tests/test_gpu_render_parity.py -q -x --timeout 600 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export FS4D_NO_TIME_ROWS=1; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ab_rows_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_rows_$v.json'));print('no_rows=$v', round(d['value'],1), d['stage_ms'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:hexplane -c 5 --csv --log-file gpurun_out/ab_rows_ncu_$v.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
  grep -E "hexplane" gpurun_out/ab_rows_ncu_$v.csv | tail -3 | cut -c1-400
done
