#!/bin/bash
# ncu launch list (time + DRAM bytes per launch) of one measured round trip: tools/prof_launches.sh TAG SHAPE DTYPE
O=gpurun_out/$1; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_$2_$3.csv python tools/prof_one.py $2 $3 > $O/ncu_$2_$3.log 2>&1
python tools/ncu_summary.py $O/launches_$2_$3.csv 1 200 > $O/launches_$2_$3.summary.txt 2>&1
grep -A40 "^total" $O/launches_$2_$3.summary.txt | head -14
