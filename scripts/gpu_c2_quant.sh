#!/bin/bash
# C2 row-quantisation sweep: PSO/Ackley dim 1000 at populations that are whole multiples of
# the resident warp count (148 SMs x 2 CTAs x 8 warps = 2368) and at C2's 10,000.
mkdir -p gpurun_out
for p in 2368 4736 7104 9472 10000 11840 14208; do
  timeout 300 python bench.py --config C2 --pop $p --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/c2q_$p.json 2> gpurun_out/c2q_$p.err
done
