# r02w: SplitMix (the reference's own stream, the drop-in default) on the headline and d=3; ncu of the headline in SplitMix mode
set -x
mkdir -p gpurun_out
for w in msc_d5 msc_d3; do
  timeout 600 python bench.py --workload $w --rng splitmix --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/bench_r02w_${w}_splitmix.json 2>> gpurun_out/bench_r02w.err
done
NK=$(python -c "import json;print(json.load(open('gpurun_out/bench_r02w_msc_d5_splitmix.json'))['config']['narrow_kn'])")
SEC=$(python bench.py --narrow-k $NK --print-sections 2>/dev/null | tail -1)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"(narrow|wide)_kernel" -s $((3 * SEC)) -c $SEC \
  -o gpurun_out/prof_r02w_splitmix python bench.py --rng splitmix --narrow-k $NK --steps 1 --warmup 3 --shots-per-step 4194304 --fixed-batch \
  --no-cpu-baseline --e2e-waves 1 > gpurun_out/ncu_full_r02w.log 2>&1
