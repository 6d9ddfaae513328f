#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python scripts/sanitize_run.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
