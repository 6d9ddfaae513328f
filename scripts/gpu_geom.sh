#!/bin/bash
# Geometry sweep: EVOX_GEOM forces 3 = 4 lanes/row, 0 = 8 lanes/row, 1 = warp/row, 2 = CTA/row.
mkdir -p gpurun_out
CFGS=${CFGS:-"C4g C4r D1"}
for g in base ${GEOMS:-3 0 1}; do
  for c in $CFGS; do
    if [ "$g" == "base" ]; then unset EVOX_GEOM; else export EVOX_GEOM=$g; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/geom_${g}_$c.json 2> gpurun_out/geom_${g}_$c.err
  done
done
unset EVOX_GEOM
