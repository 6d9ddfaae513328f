#!/bin/bash
# evox_eval bench lines: each function at the H and C5 shapes, 1 GPU.
mkdir -p gpurun_out
for fn in sphere ackley rastrigin griewank rosenbrock; do
  for s in EH E5; do
    timeout 300 python bench.py --config $s-$fn --steps 20 --warmup 3 > gpurun_out/ev_bench_$s-$fn.json 2> gpurun_out/ev_bench_$s-$fn.err
  done
done
