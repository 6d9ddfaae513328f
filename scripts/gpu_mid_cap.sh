#!/bin/bash
# Where does the persistent kernel stop paying? A/B at larger populations (EVOX_MID_MAX).
mkdir -p gpurun_out
for rep in 1 2; do
for v in mid nomid; do
  if [ $v == mid ]; then export EVOX_MID_MAX=2000000000; else unset EVOX_MID_MAX; fi
  for c in C4g C4r; do
    timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap_${v}_${c}_$rep.json 2> gpurun_out/cap_${v}_${c}_$rep.err
  done
  timeout 300 python bench.py --config C2 --pop 100000 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap_${v}_P1e5_$rep.json 2> gpurun_out/cap_${v}_P1e5_$rep.err
  timeout 300 python bench.py --config H --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cap_${v}_H_$rep.json 2> gpurun_out/cap_${v}_H_$rep.err
done
done
