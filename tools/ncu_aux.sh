#!/bin/bash
# ncu --set full of the level-L Thomas passes, recompose interpolation and assembly (warm round trip)
TAG=${1:-aux}; DT=${2:-f64}
O=gpurun_out/$TAG; mkdir -p $O
P="python tools/prof_one.py 1025x1025x1025 $DT"
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $N -k regex:"thomas_lines.*int.33" -s 4 -c 2 -o $O/thomas_strided_$DT $P > $O/ncu_ts.log 2>&1
timeout 600 $N -k regex:"thomas_rows.*int.17" -s 2 -c 1 -o $O/thomas_rows_$DT $P > $O/ncu_tr.log 2>&1
timeout 600 $N -k regex:"k_interp_rec" -s 11 -c 1 -o $O/interp_$DT $P > $O/ncu_ir.log 2>&1
timeout 600 $N -k regex:"k_scatter_even" -s 19 -c 1 -o $O/scatter_$DT $P > $O/ncu_sc.log 2>&1
echo done
