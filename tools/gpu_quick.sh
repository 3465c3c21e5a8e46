#!/bin/bash
# quick GPU iteration: given pytest selection + bench configs (dev aid)
# usage: tools/gpu_quick.sh TAG "PYTEST_ARGS" "CONFIGS..."
TAG=${1:-quick}; O=gpurun_out/$TAG; mkdir -p $O
if [ -n "$2" ]; then timeout 1200 python -m pytest $2 -x -q -rs > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -15 $O/pytest.log; fi
for c in $3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python - "$O" "$c" <<'PY'
import json, sys
o, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f'{o}/bench_{c}.json').read().strip().splitlines()[-1])
    print(c, d['value'], 'GB/s', d['ms_per_step'], 'ms', 'rt_err', '%.2e' % d['roundtrip_rel_err'])
    print('   ', {k: round(v['ms_per_step'], 3) for k, v in d['kernels'].items()})
except Exception as e:
    print(c, 'FAILED', e); print(open(f'{o}/bench_{c}.err').read()[-2500:])
PY
done
