#!/bin/bash
# r02bar1: in-place compaction with one barrier per round (GS_COMPACT_1BAR) vs the same source without it
mkdir -p gpurun_out
TAG=r02bar1 R=3 bash scripts/gpu_ab2.sh
TAG=r02bar1_grown R=2 bash scripts/gpu_ab2.sh --workload msc_d5_grown
TAG=r02bar1_c4 R=2 bash scripts/gpu_ab2.sh --workload config4_n32_t24
GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_bar1.so timeout 1500 python -m pytest tests -m gpu -x -q \
  > gpurun_out/r02bar1_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02bar1_pytest_gpu.log
