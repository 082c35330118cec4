#!/bin/bash
# Round-end pass: a last compile-time A/B (blend Gaussian group size), the
# default build restored, then the full evidence refresh (tools/gpu_profiles.sh).
mkdir -p gpurun_out
bash tools/ab_define.sh "" "-DFS4D_BLEND_BK=4" "" "-DFS4D_BLEND_BK=4" > gpurun_out/ab_bk_final.txt 2>&1
cat gpurun_out/ab_bk_final.txt
python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1; echo rebuild=$?
bash tools/gpu_profiles.sh
