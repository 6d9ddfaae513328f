#!/bin/bash
# A/B of the next-generation first-row L2 prefetch in k_pso_run_mid (EVOX_MID_PF), alternating.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mid" > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
for rep in 1 2; do
for v in pf nopf; do
  if [ $v == nopf ]; then L="$PWD/paper_2301_12457_b200/variants/libevox_nopf.so"; else L=""; fi
  for p in 4736 10000 14208 30000; do
    EVOX_LIB=$L timeout 300 python bench.py --config C2 --pop $p --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/pf_${v}_${p}_$rep.json 2> gpurun_out/pf_${v}_${p}_$rep.err
  done
done
done
