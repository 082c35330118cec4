#!/bin/bash
# Frames-in-flight scheduling A/B: stream priorities (FS4D_SEQ_PRIO) x stream count.
mkdir -p gpurun_out
for cfg in "0 3" "1 3" "0 4" "1 4" "1 3" "0 3"; do
  set -- $cfg
  FS4D_SEQ_PRIO=$1 FS4D_SEQ_STREAMS=$2 timeout 300 python bench.py --no-cpu > gpurun_out/ap.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ap.json').read().strip().splitlines()[-1]);print('prio=$1 streams=$2', round(d['value'],1))"
done
