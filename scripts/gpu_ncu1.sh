#!/bin/bash
# One ncu --set full capture of the sampling kernel on the default bench
# workload (TAG names the outputs; extra args go to bench.py).
mkdir -p gpurun_out
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s 12 -c 4 \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG}.log
