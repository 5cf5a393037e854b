#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --shots-per-step 262144 --no-cpu-baseline > gpurun_out/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 \
  -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 1 --shots-per-step 262144 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
