#!/bin/bash
# r02stz: predicated store pair for pruned chi entries (GS_BF_STZ) vs HEAD --
# headline A/B interleaved (3 rounds), then d=3 and the grown proxy, then the
# GPU suite on the variant
mkdir -p gpurun_out
TAG=r02stz R=3 bash scripts/gpu_ab2.sh
TAG=r02stz_d3 R=2 bash scripts/gpu_ab2.sh --workload msc_d3
TAG=r02stz_grown R=2 bash scripts/gpu_ab2.sh --workload msc_d5_grown
GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_stz.so timeout 1500 python -m pytest tests -m gpu -x -q \
  > gpurun_out/r02stz_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02stz_pytest_gpu.log
