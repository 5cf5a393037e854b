# r02hh: fused T pairs without the gate-1 count: all GPU tests + A/B vs HEAD (Philox headline, d=3, grown)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02hh.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02hh.log
TAG=r02hh bash scripts/gpu_ab_tree.sh
for w in msc_d3 msc_d5_grown config1; do
  (cd _ab_base && timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > ../gpurun_out/ab_r02hh_base_$w.json 2>/dev/null)
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ab_r02hh_new_$w.json 2>/dev/null
  echo "$w base $(python -c "import json;print(json.load(open('gpurun_out/ab_r02hh_base_$w.json'))['value'])") new $(python -c "import json;print(json.load(open('gpurun_out/ab_r02hh_new_$w.json'))['value'])")" >> gpurun_out/ab_r02hh.txt
done
cat gpurun_out/ab_r02hh.txt
