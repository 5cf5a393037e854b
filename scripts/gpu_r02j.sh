# r02j: narrow chi limit 5 (new default) + no-span pivot part-pass: GPU tests, smoke,
# A/B of KN / narrow split / narrow blocks on the headline, KN 4 vs 5 on d=3 and the grown proxy
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02j.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02j.log
TAG=r02j R=2 bash scripts/gpu_ab2.sh
for w in msc_d3 msc_d5_grown; do
  for v in kn4 kn5; do
    GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_$v.so timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-waves 1 > gpurun_out/ab_r02j_${w}_$v.json 2>> gpurun_out/ab_r02j.err
    echo "$w $v $(python -c "import json;print(json.load(open('gpurun_out/ab_r02j_${w}_$v.json'))['value'])" 2>&1)" >> gpurun_out/ab_r02j.txt
  done
done
for nt in "56 16" "48 24" "24 24" "64 32"; do
  timeout 300 python scripts/c4_point.py $nt --shots 20000 >> gpurun_out/c4_r02j.txt 2>> gpurun_out/c4_r02j.err
done
