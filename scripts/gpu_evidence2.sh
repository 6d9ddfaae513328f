#!/bin/bash
# tests + smoke + bench lines (with cpu_baseline) for every config; N=2 flows on one GPU
mkdir -p gpurun_out
bash scripts/gpu_check.sh quick
for c in H C1 C2 C3 C4g C4r C5 D1 D2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
done
for c in C3 D1; do
  EVOX_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29520 + RANDOM % 100)) bench.py --gpus 2 --config $c --pop 20000 --steps 4 \
    --warmup 3 --no-cpu-baseline > gpurun_out/same2_$c.json 2> gpurun_out/same2_$c.err
done
