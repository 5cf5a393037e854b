#!/bin/bash
# A/B of the working tree against a committed revision checked out as a git
# worktree in _ab_base/ (git-ignored, travels with the gpurun snapshot):
#   git worktree add _ab_base HEAD && (cd _ab_base && python -c "import __graft_entry__ as g; g.build()")
#   gpurun -- 'TAG=x bash scripts/gpu_ab_tree.sh'
# Unlike gpu_ab.sh (library variants under one Python compiler) this also
# compares compiler (op-stream) changes.
mkdir -p gpurun_out
TAG=${TAG:-abt}
for i in 1 2; do
  (cd _ab_base && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > ../gpurun_out/ab_${TAG}_base_$i.json 2>/dev/null)
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ab_${TAG}_new_$i.json 2>/dev/null
done
for f in gpurun_out/ab_${TAG}_*.json; do
  echo "$f $(python -c "import json;print(json.load(open('$f'))['value'])" 2>&1)"
done | tee gpurun_out/ab_${TAG}.txt
