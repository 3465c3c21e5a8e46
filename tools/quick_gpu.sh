#!/bin/bash
# quick GPU check: parity suite + brief bench of the given configs (dev aid)
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/quick/pytest.log 2>&1; tail -30 gpurun_out/quick/pytest.log | grep -v "^$" | tail -25
for c in "$@"; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/quick/bench_$c.json 2> gpurun_out/quick/bench_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/quick/bench_{c}.json').read().strip().splitlines()[-1])
    print(c, d['value'], 'GB/s', d['ms_per_step'], 'ms', 'rt_err', '%.2e' % d['roundtrip_rel_err'])
    print('   ', {k: round(v['ms_per_step'], 3) for k, v in d['kernels'].items()})
except Exception as e:
    print(c, 'FAILED', e); print(open(f'gpurun_out/quick/bench_{c}.err').read()[-1500:])
PY
done
