#!/bin/bash
# ncu --set full with source attribution for each CFG:KERNEL:POP, exported as CSV (rep dropped)
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read CFG KRE POP <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
      -o gpurun_out/sp_$CFG -f python bench.py --config $CFG --pop $POP --steps 2 --warmup 3 \
      --no-cpu-baseline --e2e-steps 1 > gpurun_out/sp_$CFG.log 2>&1
  ncu -i gpurun_out/sp_$CFG.ncu-rep --page source --csv --print-source sass > gpurun_out/sp_src_$CFG.csv 2>&1
  python scripts/ncu_summary.py gpurun_out/sp_$CFG.ncu-rep > gpurun_out/sp_sum_$CFG.txt 2>&1
  rm -f gpurun_out/sp_$CFG.ncu-rep
done
