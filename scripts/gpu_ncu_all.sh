# One ncu --set full capture of the generation kernel of every bench config (raw CSV exported on
# the box; summarised here with scripts/ncu_summary.py), plus the H launch list.
#   bash scripts/gpu_ncu_all.sh [tag]   -> gpurun_out/ncu_<tag>_<cfg>_raw.csv, launches_<tag>_H.csv
tag=${1:-r02}
mkdir -p gpurun_out
for ck in H:k_pso_gen_wave C3:k_cso_gen C4g:k_pso_gen_flat C4r:k_pso_gen_flat \
          C5:k_pso_gen_wave D1:k_de_gen_flat D2:k_de_gen EH-ackley:k_eval E5-griewank:k_eval; do
  c=${ck%%:*}; k=${ck#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o /tmp/prof_${tag}_$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 1 --sustained-s 0 > gpurun_out/ncu_${tag}_$c.log 2>&1
  ncu -i /tmp/prof_${tag}_$c.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_${c}_raw.csv 2>&1
  echo "$c rc=$? $(wc -c < gpurun_out/ncu_${tag}_${c}_raw.csv)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${tag}_H.csv python bench.py --config H --steps 2 --warmup 1 \
  --no-cpu-baseline --e2e-steps 1 --sustained-s 0 > gpurun_out/launches_${tag}_H.log 2>&1
echo "launches rc=$?"
