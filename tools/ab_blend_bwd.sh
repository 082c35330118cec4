for px in 1 2 4; do
  FS4D_BLEND_BWD_PX=$px timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"blend_bwd" -c 4 --csv --log-file gpurun_out/bb_$px.csv python bench.py --workload train --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
  echo px=$px; python tools/ncu_summary.py launches gpurun_out/bb_$px.csv | tail -1
done
