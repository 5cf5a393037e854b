# r02bb: sanitizers on the register-state build + the config-4 grid + BASELINE configs on HEAD
set -x
mkdir -p gpurun_out
TAG=r02bb bash scripts/gpu_sanitize.sh
timeout 1500 python scripts/config4_sweep.py --shots 50000 --out gpurun_out/config4_sweep_r02bb.jsonl > gpurun_out/config4_sweep_r02bb.log 2>&1
for w in msc_d3 msc_d5_grown config1 injection_d3 msc_d5_2check; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r02bb_$w.json 2>> gpurun_out/bench_r02bb.err
done
