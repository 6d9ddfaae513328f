#!/bin/bash
# C2 row quantisation: 3 resident CTAs/SM (80-register cap) for the persistent kernel, A/B.
mkdir -p gpurun_out
for rep in 1 2; do
for v in base minb3 minb3u3; do
  if [ $v == base ]; then L=""; else L="$PWD/paper_2301_12457_b200/variants/libevox_$v.so"; fi
  for p in 7104 10000 14208; do
    EVOX_LIB=$L timeout 300 python bench.py --config C2 --pop $p --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mb_${v}_${p}_$rep.json 2> gpurun_out/mb_${v}_${p}_$rep.err
  done
done
done
