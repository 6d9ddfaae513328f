#!/bin/bash
# Grid sweep: persistent (unset) vs EVOX_NP=k waves / 0 = one CTA per row unit.
mkdir -p gpurun_out
CFGS=${CFGS:-"H C2 C3 C4g C4r C5 D1 D2"}
for np in base ${NPS:-0 4}; do
  for c in $CFGS; do
    if [ "$np" == "base" ]; then unset EVOX_NP; else export EVOX_NP=$np; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/np_${np}_$c.json 2> gpurun_out/np_${np}_$c.err
  done
done
unset EVOX_NP
