#!/bin/bash
# compute-sanitizer over the streaming / face / level kernels on small shapes (dev aid)
O=gpurun_out/${1:-san}; mkdir -p $O
export HGR_STREAM_MIN=0  # every level through the streaming passes (fp64 default: >= 2^20 nodes)
for t in memcheck synccheck racecheck; do
  for spec in 17x257x129:f64 17x257x129:f32 33x129x65:f64 65x65x65:f32; do
    IFS=: read shp dt <<< "$spec"
    timeout 600 compute-sanitizer --tool $t --print-limit 10 python tools/dbg_inplace.py $shp $dt > $O/${t}_${shp}_${dt}.log 2>&1
    echo "$t $shp $dt rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $O/${t}_${shp}_${dt}.log | tr '\n' ' ')"
  done
done
