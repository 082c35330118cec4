for d in "" "-DFS4D_EMIT_THREADS=256" "-DFS4D_EMIT_THREADS=1024"; do
  FS4D_EXTRA_NVCC="$d" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/l.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "[$d]"; python tools/ncu_summary.py launches gpurun_out/l.csv | grep "emit\|tile_sort"
done
