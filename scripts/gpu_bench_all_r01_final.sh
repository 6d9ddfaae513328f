#!/bin/bash
# Closing refresh of every bench line (1 GPU) after the persistent-kernel and best() changes.
mkdir -p gpurun_out
for c in H C1 C2 C3 C4g C4r C5 D1 D2; do
  timeout 600 python bench.py --config $c > gpurun_out/fb_$c.json 2> gpurun_out/fb_$c.err
done
