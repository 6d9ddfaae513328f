#!/bin/bash
# Round-1 evidence for the persistent mid-size kernel: GPU suite, C2 bench line, ncu.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ev_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/ev_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$? >> gpurun_out/ev_smoke.log
timeout 600 python bench.py --config C2 > gpurun_out/ev_C2.json 2> gpurun_out/ev_C2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/ev_launches_C2.csv python bench.py --config C2 --steps 4 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/ev_launches_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pso_run_mid -s 1 -c 1 \
    -o gpurun_out/prof_C2mid -f python bench.py --config C2 --steps 4 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_C2mid.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_C2mid.log
