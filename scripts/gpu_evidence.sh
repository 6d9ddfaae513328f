#!/bin/bash
# Evidence for profiles/: bench lines (with cpu_baseline) for every config, the H launch list,
# and one ncu --set full capture per listed config.
mkdir -p gpurun_out
for c in H C1 C2 C3 C4g C4r C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/ev_launches_H.csv python bench.py --config H --steps 4 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for spec in H:k_pso_gen C4g:k_pso_gen C3:k_cso_gen C5:k_pso_gen; do
  IFS=: read CFG KRE <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
      -o gpurun_out/ev_prof_$CFG -f python bench.py --config $CFG --steps 2 --warmup 3 \
      --no-cpu-baseline --e2e-steps 1 > gpurun_out/ev_prof_$CFG.log 2>&1
  python scripts/ncu_summary.py gpurun_out/ev_prof_$CFG.ncu-rep > gpurun_out/ev_ncu_$CFG.txt 2>&1
  ncu -i gpurun_out/ev_prof_$CFG.ncu-rep --page raw --csv > gpurun_out/ev_ncu_raw_$CFG.csv 2>/dev/null
  [ "$CFG" != "H" ] && rm -f gpurun_out/ev_prof_$CFG.ncu-rep
done
