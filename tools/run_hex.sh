timeout 900 python -m pytest tests/test_gpu_deform_parity.py tests/test_gpu_train.py -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error" gpurun_out/gpu_tests.log | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hexplane_bwd|mlp_bwd|blend_bwd|preprocess_bwd|passthrough" -c 20 --csv --log-file gpurun_out/hex_launches.csv python bench.py --workload train --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu=$?
python tools/ncu_summary.py launches gpurun_out/hex_launches.csv
