#!/bin/bash
# Round-1 closing evidence: GPU suite, smoke, default bench lines (H, C2), C2 ncu of the final kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$? >> gpurun_out/fin_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fin_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/fin_gpu_tests.log
python bench.py > gpurun_out/fin_H.json 2> gpurun_out/fin_H.err
timeout 600 python bench.py --config C2 > gpurun_out/fin_C2.json 2> gpurun_out/fin_C2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pso_run_mid -s 1 -c 1 \
    -o gpurun_out/prof_C2mid_fin -f python bench.py --config C2 --steps 4 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_C2mid_fin.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_C2mid_fin.log
