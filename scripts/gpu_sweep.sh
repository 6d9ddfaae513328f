timeout 1200 python scripts/sweep.py --steps 20 > gpurun_out/r02_sweeps.txt 2>&1; echo sweep_rc=$?
cp profiles/r02_sweeps.jsonl gpurun_out/ 2>/dev/null
bash scripts/gpu_ncu.sh H H k_pso_gen
bash scripts/gpu_ncu.sh C5 C5 k_pso_gen_wave
bash scripts/gpu_ncu.sh D1 D1 k_de_gen
du -sh gpurun_out
