#!/bin/bash
# Refresh the committed evidence: tests, smoke, benches, launch lists, ncu --set full of the top kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --workload train --steps 5 --warmup 3 --no-cpu > gpurun_out/train.json 2>&1; echo train=$?
timeout 600 python bench.py --workload fine --steps 5 --warmup 3 --no-cpu > gpurun_out/fine.json 2>&1; echo fine=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/train_launches.csv python bench.py --workload train --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu_train=$?
bash tools/ncu_full_render.sh; bash tools/ncu_full_train.sh; for k in; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k[<(]" -s 3 -c 1 -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "full $k rc=$?"
done
