bash tools/ab_define.sh "-DFS4D_GATHER_MINB=9" "" "-DFS4D_GATHER_MINB=9" ""
bash tools/ab_carve.sh
