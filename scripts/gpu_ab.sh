#!/bin/bash
# A/B the prebuilt variants (scripts/build_variants.sh) on one GPU:
#   TAG=x bash scripts/gpu_ab.sh [extra bench args]
mkdir -p gpurun_out
TAG=${TAG:-ab}
for so in paper_2512_23037_b200/variants/libgstab_*.so; do
  name=$(basename $so .so)
  GSTAB_LIB=$PWD/$so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" \
    > gpurun_out/ab_${TAG}_${name}.json 2>> gpurun_out/ab_${TAG}.err
  echo "$name $(python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_${name}.json'));print(d['value'])" 2>&1)" >> gpurun_out/ab_${TAG}.txt
done
cat gpurun_out/ab_${TAG}.txt
