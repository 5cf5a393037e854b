# r02f: block form on global chi -- ping-pong buffers, fused span pivot +
# compaction, unrolled read-only passes: parity tests + config-4 A/B vs _ab_base
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_r02f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02f.log
for nt in "56 16" "48 24" "40 24" "24 24" "64 24" "48 32"; do
  timeout 300 python _ab_base/scripts/c4_point.py $nt --shots 20000 | sed 's/^/base /' >> gpurun_out/c4_r02f.txt 2>> gpurun_out/c4_r02f.err
  timeout 300 python scripts/c4_point.py $nt --shots 20000 | sed 's/^/new  /' >> gpurun_out/c4_r02f.txt 2>> gpurun_out/c4_r02f.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 \
  -o gpurun_out/prof_r02f_c4_n48_t24 python scripts/c4_point.py 48 24 --shots 4000 --warm 0 > gpurun_out/ncu_r02f.log 2>&1
