#!/bin/bash
# One GPU pass: gpu tests, smoke, render bench, train bench, launch lists.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -c 3000 gpurun_out/bench.json
timeout 600 python bench.py --workload train --steps 5 --warmup 3 --no-cpu > gpurun_out/train.json 2> gpurun_out/train.err; echo train=$?; cat gpurun_out/train.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$?; cat gpurun_out/ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu=$?
python tools/ncu_summary.py launches gpurun_out/launches.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/train_launches.csv python bench.py --workload train --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_train.log 2>&1; echo ncu_train=$?
python tools/ncu_summary.py launches gpurun_out/train_launches.csv
