#!/bin/bash
# ncu --set full captures of the hot kernels on one warm 1025^3 round trip (dev aid).
# usage: tools/ncu_full.sh TAG [dtype]
TAG=${1:-full}; DT=${2:-f64}
O=gpurun_out/$TAG; mkdir -p $O
P="python tools/prof_one.py 1025x1025x1025 $DT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level_fused -s 4 -c 4 -o $O/level_$DT $P > $O/ncu_level.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_thomas_strided|k_thomas_rows" -s 12 -c 3 -o $O/thomas_$DT $P > $O/ncu_thomas.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_interp_rec|k_scatter_even" -s 20 -c 20 -o $O/interp_$DT $P > $O/ncu_interp.log 2>&1
echo done
