#!/bin/bash
# build a measurement variant: one source recompiled with defines, linked with build/ objects
# usage: var_build.sh <name> <src.cu> DEF=1 ...
cd /root/repo/paper_2301_12457_b200
name=$1; src=$2; shift 2
mkdir -p /tmp/var_$name variants
D=""; for d in "$@"; do D="$D -D$d"; done
base=$(basename $src .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-Wall -I ../include -I csrc -I /usr/include $D -c csrc/$src -o /tmp/var_$name/$base.o || exit 1
objs=""
for o in pso_kernels cso_kernels de_kernels common_kernels evox_api nccl_dl; do
  if [ $o == $base ]; then objs="$objs /tmp/var_$name/$o.o"; else objs="$objs build/$o.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/libevox_$name.so $objs -ldl -lpthread && echo built $name
