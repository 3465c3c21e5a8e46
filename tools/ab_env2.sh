#!/bin/bash
# two-knob sweep on one box: tools/ab_env2.sh VAR1 "v..." VAR2 "w..." config...
V1=$1; A1=$2; V2=$3; A2=$4; shift 4
for c in "$@"; do
  for a in $A1; do for b in $A2; do
    export $V1=$a $V2=$b
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c $V1=$a $V2=$b', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done; done
done
