# Ablation of the fused PSO generation at H (measurement builds in variants/, EVOX_ABL bits:
# 1 no Philox, 2 no fitness terms, 4 no gbest load; pf0 = no L2 bulk prefetch)
out=gpurun_out/r02_abl.txt; : > $out
for v in base a1 a2 a4 a3 a7 pf0; do
  if [ $v == base ]; then L=""; else L="$PWD/paper_2301_12457_b200/variants/libevox_$v.so"; fi
  r=$(EVOX_LIB=$L timeout 300 python bench.py --config H --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1)
  echo "H $v $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"],2), round(r["frac"],4), r.get("kernel_ms"))' 2>&1)" >> $out
done
for v in base pf0; do
  if [ $v == base ]; then L=""; else L="$PWD/paper_2301_12457_b200/variants/libevox_$v.so"; fi
  EVOX_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_pso_gen -s 3 -c 2 python bench.py --config H --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_ncu_H_$v.txt 2>&1
done
cat $out
