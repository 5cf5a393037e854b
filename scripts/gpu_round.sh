#!/bin/bash
# One gpurun call: build check, GPU tests, smoke, bench, ncu evidence.
#   TAG=r01b bash scripts/gpu_round.sh [--no-tests] [--no-ncu]
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [[ " $* " != *" --no-tests "* ]]; then
  timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?" >> gpurun_out/bench_${TAG}.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 6 > gpurun_out/bench_ref_${TAG}.json 2>> gpurun_out/bench_${TAG}.err
for v in ${VARIANTS:-}; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${v//,/ } > "gpurun_out/bench_${TAG}_var_${v}.json" 2>> gpurun_out/bench_${TAG}.err
done
if [[ " $* " != *" --no-ncu "* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench_${TAG}.json 2>&1
  # one step of 2^22 shots = one chunk: its section launches, after 3 warm-up steps
  SEC=$(python bench.py --print-sections 2>/dev/null | tail -1)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s $((3 * SEC)) -c $SEC \
    -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --shots-per-step 4194304 --fixed-batch --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG}.log
fi
