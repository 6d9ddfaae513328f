#!/bin/bash
# Bench the tuning variants in paper_2301_12457_b200/variants/ on several configs.
mkdir -p gpurun_out
CFGS=${CFGS:-"H C4g C5 C3"}
for v in base $VARIANTS; do
  for c in $CFGS; do
    if [ "$v" == "base" ]; then L=""; else L="$PWD/paper_2301_12457_b200/variants/libevox_$v.so"; fi
    EVOX_LIB=$L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/${PREFIX}var_${v}_$c.json 2> gpurun_out/${PREFIX}var_${v}_$c.err
  done
done
