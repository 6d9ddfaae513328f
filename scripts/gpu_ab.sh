# same-box A/B of measurement builds in paper_2301_12457_b200/variants/ (built by
# scripts/var_build.sh): bash scripts/gpu_ab.sh "<configs>" "<base|variant names>" [reps]
# same-box A/B of library variants: bash scripts/gpu_r02_ab.sh "<configs>" "<variants>" [reps]
out=gpurun_out/r02_ab.txt; : > $out
for rep in $(seq 1 ${3:-1}); do
for c in $1; do
  for v in $2; do
    if [ $v == base ]; then L=""; else L="$PWD/paper_2301_12457_b200/variants/libevox_$v.so"; fi
    r=$(EVOX_LIB=$L timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1)
    echo "$c $v $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"],2), round(r["frac"],4), r.get("kernel_ms"))' 2>&1)" >> $out
  done
done
done
cat $out
