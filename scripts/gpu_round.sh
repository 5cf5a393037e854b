#!/bin/bash
# One gpurun call: build check, GPU tests, smoke, bench (+ variants).
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
for v in "--chi-smem" "--dense-only" "--rng splitmix"; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $v > "gpurun_out/bench_var_${v// /_}.json" 2>> gpurun_out/bench.err
done
