#!/bin/bash
# Build compile-time variants of the sampler for on-GPU A/B runs:
#   bash scripts/build_variants.sh "NAME:-DFOO=1 -DBAR=2" ...
# -> paper_2512_23037_b200/variants/libgstab_NAME.so (use via GSTAB_LIB=...)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2512_23037_b200/variants
for spec in "$@"; do
  name=${spec%%:*}
  defs=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
    $defs -o paper_2512_23037_b200/variants/libgstab_${name}.so paper_2512_23037_b200/csrc/gs_kernels.cu &
done
wait
ls paper_2512_23037_b200/variants
