#!/bin/bash
# One GPU round: parity tests, smoke, bench, ncu launch list + full capture of the top kernel.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [quick]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
[ "$1" == "quick" ] && exit 0
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_H.json 2> gpurun_out/bench_H.err
echo "bench rc=$?" >> gpurun_out/bench_H.err
