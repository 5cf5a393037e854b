#!/bin/bash
# Build kernel variants (-D flags) side by side and bench each one.
# usage: bash scripts/gpu_variants.sh "NAME:FLAGS" ...
mkdir -p gpurun_out/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  lib=$PWD/gpurun_out/variants/lib_$name.so
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared $flags \
    -o $lib paper_2512_23037_b200/csrc/gs_kernels.cu > gpurun_out/variants/build_$name.log 2>&1
  GSTAB_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/variants/bench_$name.json 2>> gpurun_out/variants/err.log
  rm -f $lib
done
