#!/bin/bash
# Training-path GPU check: train/render/determinism/world-2 tests + the configs[4] train bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -k "world2 or train or determinism or render or headline" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --workload train --steps 10 --warmup 3 --no-cpu > gpurun_out/train.json 2> gpurun_out/train.err; echo train=$?
python -c "import json;d=json.loads(open('gpurun_out/train.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['stage_ms_per_step'])"
