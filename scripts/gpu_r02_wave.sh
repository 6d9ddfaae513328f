# A/B of the persistent generation kernel against the wave grid (k_pso_gen_wave + k_pso_fin)
out=gpurun_out/r02_wave_ab.txt; : > $out
for c in H C4g C4r C5; do
  for v in base np4 wave3 wave2 waveu3; do
    case $v in
      base) E="";; np4) E="EVOX_NP=4";; wave3) E="EVOX_WAVE=1";;
      waveu3) E="EVOX_WAVE=1 EVOX_LIB=$PWD/paper_2301_12457_b200/variants/libevox_wu3.so";;
      wave2) E="EVOX_WAVE=1 EVOX_LIB=$PWD/paper_2301_12457_b200/variants/libevox_wm2.so";;
    esac
    r=$(env $E timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1)
    echo "$c $v $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"],2), round(r["frac"],4), r.get("kernel_ms"))' 2>&1)" >> $out
  done
done
cat $out
EVOX_WAVE=1 EVOX_NO_SMALL=1 EVOX_NO_MID=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "step_parity or full_size or graphed or fused_fitness" > gpurun_out/r02_wave_pytest.log 2>&1; echo wave_pytest_rc=$?; tail -3 gpurun_out/r02_wave_pytest.log
