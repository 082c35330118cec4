#!/bin/bash
# ncu --set full of the top training-step kernels (one launch each).
mkdir -p gpurun_out
for k in k_hexplane_bwd_c32 k_blend_bwd2 k_mlp_bwd_tc k_preprocess_bwd; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^$k\$" -s 2 -c 1 -o gpurun_out/full_$k -f python bench.py --workload train --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$k.log 2>&1
  echo "$k rc=$?"
done
