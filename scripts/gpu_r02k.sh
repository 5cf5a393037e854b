# r02k: run-time narrow limit (auto-tuned per program): all GPU tests, smoke,
# bench on the headline / d=3 / grown proxy, ncu launch list + full capture
set -x
mkdir -p gpurun_out
TAG=r02k
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 12 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for w in msc_d3 msc_d5_grown config1 injection_d3; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$w.json 2>> gpurun_out/bench_$TAG.err
done
NK=$(python -c "import json;print(json.load(open('gpurun_out/bench_$TAG.json'))['config']['narrow_kn'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --narrow-k $NK --steps 2 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ncu_launch_bench_$TAG.json 2>&1
SEC=$(python bench.py --narrow-k $NK --print-sections 2>/dev/null | tail -1)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s $((3 * SEC)) -c $SEC \
  -o gpurun_out/prof_$TAG python bench.py --narrow-k $NK --steps 1 --warmup 3 --shots-per-step 4194304 --fixed-batch \
  --no-cpu-baseline --e2e-waves 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$TAG.log
