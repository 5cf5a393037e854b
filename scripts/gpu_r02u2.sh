#!/bin/bash
# r02u2: fused T-pair loop unrolled 2 (GS_BF2_UNROLL=2; 128 registers, no spills) vs HEAD
mkdir -p gpurun_out
TAG=r02u2 R=3 bash scripts/gpu_ab2.sh
TAG=r02u2_grown R=2 bash scripts/gpu_ab2.sh --workload msc_d5_grown
TAG=r02u2_d3 R=2 bash scripts/gpu_ab2.sh --workload msc_d3
GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_u2.so timeout 1500 python -m pytest tests -m gpu -x -q \
  > gpurun_out/r02u2_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02u2_pytest_gpu.log
