#!/bin/bash
# One gpurun call (round 2): build, measured ceilings, GPU tests, smoke,
# bench (+ reference arm), ncu launch list + one --set full capture.
#   TAG=r02a bash scripts/gpu_round2.sh [--no-tests] [--no-ncu] [--no-ref]
set -x
TAG=${TAG:-r02}
WL=${WL:-msc_d5}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_${TAG}.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/peaks.cu \
  && timeout 120 /tmp/peaks > gpurun_out/peaks_${TAG}.json 2>&1
if [[ " $* " != *" --no-tests "* ]]; then
  timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
fi
timeout 900 python bench.py --workload $WL --steps 5 --warmup 3 --cpu-seconds 12 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?" >> gpurun_out/bench_${TAG}.err
if [[ " $* " != *" --no-ref "* ]]; then
  timeout 600 python bench.py --workload $WL --impl reference --steps 3 --warmup 1 --cpu-seconds 12 > gpurun_out/bench_ref_${TAG}.json 2>> gpurun_out/bench_${TAG}.err
fi
if [[ " $* " == *" --torchrun2 "* ]]; then
  # the multi-rank flow (barriers, max-over-ranks timing, tuned-flag
  # broadcast, counter all-reduce) with two ranks sharing the one GPU (gloo)
  GS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --workload $WL --steps 3 --warmup 3 \
    --no-cpu-baseline --e2e-waves 1 > gpurun_out/bench_${TAG}_torchrun2.json 2>> gpurun_out/bench_${TAG}.err
fi
for v in ${VARIANTS:-}; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 ${v//,/ } > "gpurun_out/bench_${TAG}_var_${v}.json" 2>> gpurun_out/bench_${TAG}.err
done
if [[ " $* " != *" --no-ncu "* ]]; then
  # the narrow limit the bench picked, fixed for the profiled runs (the
  # tuning probe would shift the launch indices)
  NK=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['config']['narrow_kn'])" 2>/dev/null || echo 4)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --workload $WL --narrow-k $NK --steps 2 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ncu_launch_bench_${TAG}.json 2>&1
  # one step of 2^22 shots = one chunk: its section launches, after 3 warm-up steps
  SEC=$(python bench.py --workload $WL --narrow-k $NK --print-sections 2>/dev/null | tail -1)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s $((3 * SEC)) -c $SEC \
    -o gpurun_out/prof_${TAG} python bench.py --workload $WL --narrow-k $NK --steps 1 --warmup 3 --shots-per-step 4194304 --fixed-batch \
    --no-cpu-baseline --e2e-waves 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG}.log
fi
