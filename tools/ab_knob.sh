#!/bin/bash
# A/B of one environment knob on bench configs (dev aid): tools/ab_knob.sh TAG VAR "V1 V2 .." CONFIG...
TAG=$1; VAR=$2; VALS=$3; shift 3; O=gpurun_out/$TAG; mkdir -p $O
for c in "$@"; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err
  python - "$O/bench_${c}_$v.json" "$c $VAR=$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], d['value'], 'GB/s', d['ms_per_step'], 'ms rt_err %.2e' % d['roundtrip_rel_err'],
          {k: round(v['ms_per_step'], 3) for k, v in d['kernels'].items()})
except Exception as e:
    print(sys.argv[2], 'FAILED', e)
PY
done; done
