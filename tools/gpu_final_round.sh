#!/bin/bash
# end-of-round evidence (dev aid): GPU suite, smoke, launch lists, ncu full briefs,
# sanitizer, then the bench lines. usage: tools/gpu_final_round.sh TAG
TAG=${1:-final}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for spec in 1025x1025x1025:f64:1025f64 1025x1025x1025:f32:1025f32 513x513x513:f32:513f32 257x513x1025:f64:aniso_nu_f64 513x513:f64:513sq_f64; do
  IFS=: read shp dt name <<< "$spec"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/ncu_launches_$name.csv python tools/prof_one.py $shp $dt >> $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu_launches_$name.csv 1 200 > $O/ncu_launches_$name.summary.txt 2>&1
done
timeout 600 bash tools/ncu_one.sh $TAG/full_dec_f64 "k_level_fused" 0 1025x1025x1025 f64 >> $O/ncu.log 2>&1
timeout 600 bash tools/ncu_one.sh $TAG/full_dec_f32 "k_level_fused" 0 1025x1025x1025 f32 >> $O/ncu.log 2>&1
timeout 600 bash tools/ncu_one.sh $TAG/full_rec_f32 "k_level_fused" 6 1025x1025x1025 f32 >> $O/ncu.log 2>&1
timeout 600 bash tools/ncu_one.sh $TAG/full_planes_f32 "k_thomas_planes_ws" 0 1025x1025x1025 f32 >> $O/ncu.log 2>&1
timeout 600 bash tools/ncu_one.sh $TAG/full_strips_f64 "k_thomas_stream" 0 1025x1025x1025 f64 >> $O/ncu.log 2>&1
timeout 600 bash tools/ncu_one.sh $TAG/full_merge_f32 "k_merge_even" 0 1025x1025x1025 f32 >> $O/ncu.log 2>&1
python tools/ncu_brief.py $O/full_dec_f64.ncu-rep $O/full_dec_f32.ncu-rep $O/full_rec_f32.ncu-rep $O/full_planes_f32.ncu-rep $O/full_strips_f64.ncu-rep $O/full_merge_f32.ncu-rep > $O/ncu_full_brief.txt 2>&1
bash tools/san_round.sh ${TAG}_san > $O/sanitizer_summary.txt 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in 1025f64 513f32 aniso_nu_f64 513sq_f64 8193sq_f32 line_f64; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python tools/time_inplace.py 1025x1025x1025 f32 > $O/inplace.txt 2>&1; python tools/time_inplace.py 1025x1025x1025 f64 >> $O/inplace.txt 2>&1
echo done
