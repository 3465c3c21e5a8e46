#!/bin/bash
# ncu --set full of the two top-level cluster Thomas launches (dim 0, dims 1+2): tools/prof_band.sh TAG [DTYPE]
T=${1:-band_prof}; DT=${2:-f32}
mkdir -p gpurun_out/$T
bash tools/ncu_one.sh $T/full_band0_$DT "k_thomas_band" 0 1025x1025x1025 $DT
bash tools/ncu_one.sh $T/full_band1_$DT "k_thomas_band" 1 1025x1025x1025 $DT
python tools/ncu_brief.py gpurun_out/$T/full_band0_$DT.ncu-rep gpurun_out/$T/full_band1_$DT.ncu-rep > gpurun_out/$T/brief_$DT.txt 2>&1
cat gpurun_out/$T/brief_$DT.txt
