#!/bin/bash
# A/B timing on one box: default build (A) vs paper_2007_04457_b200/lib_ab/libhgr_b200.so (B),
# alternating, per config. usage: tools/ab.sh config...
B=$(pwd)/paper_2007_04457_b200/lib_ab/libhgr_b200.so
for c in "$@"; do
  for rep in 1 2; do
    for v in A B; do
      if [ $v = B ]; then export HGR_B200_LIB=$B; else unset HGR_B200_LIB; fi
      timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c $v', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
    done
  done
done
