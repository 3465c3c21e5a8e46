#!/bin/bash
# A/B of env knobs on one bench config (dev aid): tools/ab_cfg.sh CONFIG "CFG1" "CFG2" ...
C=$1; shift
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --config $C --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$C $cfg', d['ms_per_step'], {k: round(v['ms_per_step'], 3) for k, v in d['kernels'].items()})"
done
