#!/bin/bash
# ncu --set full of one kernel launch: tools/ncu_one.sh OUT REGEX SKIP SHAPE DTYPE
mkdir -p $(dirname gpurun_out/$1)
ncu --set full --clock-control none --profile-from-start off --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 -o gpurun_out/$1 python tools/prof_one.py $4 $5 > gpurun_out/$1.log 2>&1
tail -n 3 gpurun_out/$1.log
