#!/bin/bash
# ncu --set full of the level-L fused kernels (decompose + recompose mode) of a warm round trip
TAG=${1:-lvl}; DT=${2:-f64}
O=gpurun_out/$TAG; mkdir -p $O
P="python tools/prof_one.py 1025x1025x1025 $DT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level_fused -s 12 -c 1 -o $O/dec_$DT $P > $O/ncu_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level_fused -s 18 -c 1 -o $O/rec_$DT $P > $O/ncu_rec.log 2>&1
echo done
