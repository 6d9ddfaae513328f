#!/bin/bash
# Bench lines for every BASELINE config (1 GPU) + full ncu capture of the headline kernel.
mkdir -p gpurun_out
for c in H C1 C2 C3 C4g C4r C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ "$1" == "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:k_pso_gen -s 3 -c 1 \
      -o gpurun_out/prof_Hfull -f python bench.py --config H --steps 2 --warmup 3 \
      --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_Hfull.log 2>&1
fi
