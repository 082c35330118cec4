#!/bin/bash
# ncu --set full of the top render kernels (one launch each, after warm-up).
# usage: bash tools/ncu_full_render.sh [kernel-name ...]   (default: the render kernels)
mkdir -p gpurun_out
KS="$*"
[ -z "$KS" ] && KS="k_blend k_mlp_tc_2s k_hexplane_latent_c32t k_preprocess k_tile_sort k_emit_partition"
for k in $KS; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^$k\$" -s 3 -c 1 -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$k.log 2>&1
  echo "full $k rc=$? $(ls gpurun_out/full_$k.ncu-rep 2>/dev/null)"
done
