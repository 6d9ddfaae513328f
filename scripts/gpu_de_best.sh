#!/bin/bash
# DE best() without the population-wide gather: DE GPU tests + D1/D2 lines (e2e).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_de.py -x -q > gpurun_out/deb_tests.log 2>&1; echo rc=$? >> gpurun_out/deb_tests.log
for c in D1 D2; do timeout 600 python bench.py --config $c > gpurun_out/deb_$c.json 2> gpurun_out/deb_$c.err; done
