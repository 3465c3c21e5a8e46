#!/bin/bash
# run bench configs and print value / ms / per-kernel ms (dev aid)
for c in "$@"; do
python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c', d['value'], 'GB/s', d['ms_per_step'], 'ms', 'rt_err', '%.2e' % d['roundtrip_rel_err'])
print('   ', {k: round(v['ms_per_step'], 3) for k, v in d['kernels'].items()})"
done
