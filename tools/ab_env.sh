#!/bin/bash
# A/B of an environment knob on one box: tools/ab_env.sh VAR "v1 v2 ..." config...
VAR=$1; VALS=$2; shift 2
for c in "$@"; do
  for v in $VALS; do
    export $VAR=$v
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c $VAR=$v', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
done
