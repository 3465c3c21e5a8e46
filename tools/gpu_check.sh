#!/bin/bash
# GPU check: parity suite, smoke, default bench line (dev aid). usage: tools/gpu_check.sh TAG
TAG=${1:-check}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/bench_default.err
tail -5 $O/pytest_gpu.log; tail -2 $O/smoke.log; tail -c 600 $O/bench_default.json
