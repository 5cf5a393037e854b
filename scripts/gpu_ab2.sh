#!/bin/bash
# A/B the prebuilt variants (scripts/build_variants.sh), interleaved, R rounds:
#   TAG=x R=2 bash scripts/gpu_ab2.sh [extra bench args]
mkdir -p gpurun_out
TAG=${TAG:-ab}
for r in $(seq ${R:-2}); do
  for so in paper_2512_23037_b200/variants/libgstab_*.so; do
    name=$(basename $so .so)
    GSTAB_LIB=$PWD/$so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 "$@" \
      > gpurun_out/ab_${TAG}_${name}_$r.json 2>> gpurun_out/ab_${TAG}.err
    echo "$name $r $(python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_${name}_$r.json'));print(d['value'])" 2>&1)" >> gpurun_out/ab_${TAG}.txt
  done
done
cat gpurun_out/ab_${TAG}.txt
