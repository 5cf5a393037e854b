#!/bin/bash
# r02sgn: reduced-form T sign applied to the ss operand once per sign class
# (GS_SGN_OPERAND) vs HEAD and vs the same source without the flag; then the
# GPU suite on the variant
mkdir -p gpurun_out
TAG=r02sgn R=3 bash scripts/gpu_ab2.sh
TAG=r02sgn_grown R=2 bash scripts/gpu_ab2.sh --workload msc_d5_grown
GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_sgn.so timeout 1500 python -m pytest tests -m gpu -x -q \
  > gpurun_out/r02sgn_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02sgn_pytest_gpu.log
