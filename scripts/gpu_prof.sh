#!/bin/bash
# ncu evidence for the dominant kernel (1 GPU): launch list + one --set full capture.
# Usage: bash scripts/gpu_prof.sh <config> <pop> <kernel-regex> <tag>
CFG=${1:-H}; POP=${2:-250000}; KRE=${3:-k_pso_gen}; TAG=${4:-H}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --config $CFG --steps 4 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_${TAG}.bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
    -o gpurun_out/prof_${TAG} -f python bench.py --config $CFG --pop $POP --steps 2 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_${TAG}.log
