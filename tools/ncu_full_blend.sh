#!/bin/bash
# ncu --set full of the top render kernels (one launch each) for the profiles.
mkdir -p gpurun_out
for k in k_blend k_mlp_tc_2s k_hexplane_latent_c32t k_tile_sort k_emit_partition k_preprocess; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$k.log 2>&1
  echo "$k rc=$?"
done
