#!/bin/bash
# A/B of streaming-IPK knobs on the default bench (dev aid): tools/ab_stream.sh "CFG1" "CFG2" ...
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', d['ms_per_step'], d['kernels']['thomas']['ms_per_step'])"
done
