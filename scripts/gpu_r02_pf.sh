# L2 bulk prefetch (mode A) on/off and occupancy variants of the PSO generation, per config
out=gpurun_out/r02_pf.txt; : > $out
for c in H C4g C4r C2 C5; do
  for v in base pf0 pf0np4 pf0m3 pf0u3m3 pf0u5m1; do
    E="EVOX_NO_MID=1"
    case $v in
      base) L="";; pf0) L=pf0;; pf0np4) L=pf0; E="$E EVOX_NP=4";; *) L=$v;;
    esac
    if [ -n "$L" ]; then L="$PWD/paper_2301_12457_b200/variants/libevox_$L.so"; fi
    r=$(env $E EVOX_LIB=$L timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1)
    echo "$c $v $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"],2), round(r["frac"],4), r.get("kernel_ms"))' 2>&1)" >> $out
  done
done
cat $out
