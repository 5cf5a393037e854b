#!/bin/bash
# ncu evidence: launch list of one bench command + full captures of the
# sampling kernel in the configurations named on the command line.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --shots-per-step 262144 --no-cpu-baseline > gpurun_out/ncu_launch_bench_${TAG}.json 2>&1
i=0
for v in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_$i python bench.py --steps 1 --warmup 1 --shots-per-step 262144 --no-cpu-baseline $v > gpurun_out/ncu_full_${TAG}_$i.log 2>&1
  echo "$i: $v rc=$?" >> gpurun_out/ncu_index_${TAG}.txt
  i=$((i+1))
done
