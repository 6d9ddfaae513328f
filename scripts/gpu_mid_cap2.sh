#!/bin/bash
# Persistent kernel with plain (L1-cached, coherent) G loads: tests + A/B against per-generation launches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pso" > gpurun_out/cap2_tests.log 2>&1; echo rc=$? >> gpurun_out/cap2_tests.log
export EVOX_MID_MAX=2000000000
for rep in 1 2; do
for v in mid nomid; do
  if [ $v == mid ]; then unset EVOX_NO_MID; else export EVOX_NO_MID=1; fi
  for c in C2 C4g C4r; do
    timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap2_${v}_${c}_$rep.json 2> gpurun_out/cap2_${v}_${c}_$rep.err
  done
  timeout 300 python bench.py --config C4g --pop 100000 --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap2_${v}_G1e5_$rep.json 2> gpurun_out/cap2_${v}_G1e5_$rep.err
  timeout 300 python bench.py --config H --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap2_${v}_H_$rep.json 2> gpurun_out/cap2_${v}_H_$rep.err
done
done
