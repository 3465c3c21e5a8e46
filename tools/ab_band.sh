#!/bin/bash
# A/B of the IPK strategies (HGR_THOMAS_BAND=0/1/2) on bench configs (dev aid)
TAG=${1:-ab}; shift; O=gpurun_out/$TAG; mkdir -p $O
for c in "$@"; do for m in 0 1 2; do
  HGR_THOMAS_BAND=$m timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_$m.json 2> $O/bench_${c}_$m.err
  python - "$O/bench_${c}_$m.json" "$c band=$m" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], d['value'], 'GB/s', d['ms_per_step'], 'ms rt_err %.2e' % d['roundtrip_rel_err'], 'thomas', round(d['kernels']['thomas']['ms_per_step'], 3))
except Exception as e:
    print(sys.argv[2], 'FAILED', e)
PY
done; done
