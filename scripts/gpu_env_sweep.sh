#!/bin/bash
# Env-switch sweep: VAR=name, VALS="base v1 v2 ..." (base = unset), CFGS=configs.
mkdir -p gpurun_out
for v in ${VALS:-base}; do
  for c in ${CFGS:-H}; do
    if [ "$v" == "base" ]; then unset $VAR; else export $VAR=$v; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/env_${VAR}_${v}_$c.json 2> gpurun_out/env_${VAR}_${v}_$c.err
  done
done
unset $VAR
