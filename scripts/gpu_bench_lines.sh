#!/bin/bash
# Bench lines (with cpu_baseline) for every config on 1 GPU -> gpurun_out/ev_bench_<cfg>.json
mkdir -p gpurun_out
for c in ${CFGS:-H C1 C2 C3 C4g C4r C5 D1 D2}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
done
