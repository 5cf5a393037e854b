# r02p: per-section narrow layout (kn 4 or 5 per narrow section) vs HEAD 5d32fa7:
# headline (auto), d=3 and grown proxy at forced kn=5 and auto; parity subset
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "golden or storage_modes or oracle or chunking or lane_per_shot" > gpurun_out/pytest_r02p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02p.log
for r in 1 2; do
 for w in "msc_d5" "msc_d3 --narrow-k 5" "msc_d5_grown --narrow-k 5" "msc_d3" "msc_d5_grown"; do
  n=$(echo $w | tr ' ' '_')
  (cd _ab_base && timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > ../gpurun_out/ab_r02p_base_${n}_$r.json 2>/dev/null)
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ab_r02p_new_${n}_$r.json 2>/dev/null
  echo "$n $r base $(python -c "import json;d=json.load(open('gpurun_out/ab_r02p_base_${n}_$r.json'));print(d['value'], d['config']['narrow_kn'])") new $(python -c "import json;d=json.load(open('gpurun_out/ab_r02p_new_${n}_$r.json'));print(d['value'], d['config']['narrow_kn'])")" >> gpurun_out/ab_r02p.txt
 done
done
cat gpurun_out/ab_r02p.txt
