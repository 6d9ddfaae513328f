#!/bin/bash
# Pinned single-sync best(): GPU suite + e2e lines of the small configs.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/best_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/best_gpu_tests.log
for c in C1 C2; do timeout 600 python bench.py --config $c > gpurun_out/best_$c.json 2> gpurun_out/best_$c.err; done
