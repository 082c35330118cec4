#!/bin/bash
# Quick GPU check after a kernel change: GPU tests (optionally a subset), render bench, launch list.
# usage: bash tools/gpu_quick.sh [pytest -k expr]
mkdir -p gpurun_out
KEXPR="${1:-}"
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 ${KEXPR:+-k "$KEXPR"} > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "serial", d["value_serial"]["value"], "stage_ms", d["stage_ms"], "e2e", d["e2e"]["value"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu=$?
python tools/ncu_summary.py launches gpurun_out/launches.csv | head -16
