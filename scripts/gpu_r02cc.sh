# r02cc: SplitMix fire test stepping the pre-mix counter (narrow kernel): SplitMix A/B vs HEAD + SplitMix parity tests
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_r02cc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02cc.log
TAG=r02cc_smx bash scripts/gpu_ab_tree.sh --rng splitmix
for w in msc_d3 msc_d5_grown; do
  (cd _ab_base && timeout 300 python bench.py --workload $w --rng splitmix --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > ../gpurun_out/ab_r02cc_base_$w.json 2>/dev/null)
  timeout 300 python bench.py --workload $w --rng splitmix --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ab_r02cc_new_$w.json 2>/dev/null
  echo "$w splitmix base $(python -c "import json;print(json.load(open('gpurun_out/ab_r02cc_base_$w.json'))['value'])") new $(python -c "import json;print(json.load(open('gpurun_out/ab_r02cc_new_$w.json'))['value'])")" >> gpurun_out/ab_r02cc_smx.txt
done
cat gpurun_out/ab_r02cc_smx.txt
