#!/bin/bash
# ncu --set full captures for the kernels below 80 % of the HBM peak (one GPU).
mkdir -p gpurun_out
prof() {  # config pop kernel-regex tag
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 \
    -o gpurun_out/prof_$4 -f python bench.py --config $1 --pop $2 --steps 2 --warmup 3 \
    --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_$4.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/prof_$4.log
}
prof E5-rosenbrock 10000 k_eval E5-rosenbrock
prof E5-griewank 10000 k_eval E5-griewank
prof D1 1000000 k_de_gen D1
prof C4r 1000000 k_pso_gen C4r
