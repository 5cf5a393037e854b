#!/bin/bash
# One ncu --set full capture of the sampling kernel on the default bench
# workload (TAG names the outputs; extra args go to bench.py).
mkdir -p gpurun_out
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# one step of 2^22 shots = one chunk: its section launches, after 3 warm-up steps
SEC=$(python bench.py --print-sections "$@" 2>/dev/null | tail -1)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s $((3 * SEC)) -c $SEC \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --shots-per-step 4194304 --fixed-batch --no-cpu-baseline "$@" > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG}.log
