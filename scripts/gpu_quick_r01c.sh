#!/bin/bash
# Rosenbrock interior fast path: parity subset + bench lines (1 GPU).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "rosenbrock or fused_fitness or sharded or peer" -p no:cacheprovider > gpurun_out/pytest_ros.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ros.log
for c in E5-rosenbrock EH-rosenbrock C4r; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
