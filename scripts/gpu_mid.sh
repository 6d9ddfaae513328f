#!/bin/bash
# Persistent mid-size PSO kernel: bitwise tests, PSO parity, C2 A/B, pop sweep, H unchanged.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mid or pso" > gpurun_out/mid_tests.log 2>&1; echo rc=$? >> gpurun_out/mid_tests.log
for v in mid nomid; do
  if [ $v == nomid ]; then export EVOX_NO_MID=1; else unset EVOX_NO_MID; fi
  timeout 300 python bench.py --config C2 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mid_C2_$v.json 2> gpurun_out/mid_C2_$v.err
  for p in 2368 4736 9472 14208 30000; do
    timeout 300 python bench.py --config C2 --pop $p --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mid_q_${v}_$p.json 2> gpurun_out/mid_q_${v}_$p.err
  done
done
unset EVOX_NO_MID
timeout 300 python bench.py --config H --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/mid_H.json 2> gpurun_out/mid_H.err
