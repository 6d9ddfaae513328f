#!/bin/bash
# ncu --set full of the generation kernel for several configs (1 GPU).
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read CFG POP KRE <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
      -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --pop $POP --steps 2 --warmup 3 \
      --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_$CFG.log 2>&1
done
