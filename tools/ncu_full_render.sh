#!/bin/bash
# ncu --set full of the top render kernels (one launch each, after warm-up).
mkdir -p gpurun_out
for k in k_blend k_mlp_tc_ws k_hexplane_latent_c32t k_preprocess k_tile_sort k_emit_partition; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^$k\$" -s 3 -c 1 -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$k.log 2>&1
  echo "full $k rc=$? $(ls gpurun_out/full_$k.ncu-rep 2>/dev/null)"
done
