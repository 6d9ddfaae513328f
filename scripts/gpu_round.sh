#!/bin/bash
# tests + smoke + bench lines for every config (one GPU call)
bash scripts/gpu_check.sh quick
for c in H C1 C2 C3 C4g C4r C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
