# r02h: span pivots in one pass (both outcomes) in the block form: tests + config-4 points
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_reference_semantics.py -q -x > gpurun_out/pytest_r02h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02h.log
for nt in "56 16" "48 24" "40 24" "24 24" "48 32" "32 32" "64 32"; do
  timeout 300 python scripts/c4_point.py $nt --shots 20000 >> gpurun_out/c4_r02h.txt 2>> gpurun_out/c4_r02h.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 \
  -o gpurun_out/prof_r02h_c4_n48_t24 python scripts/c4_point.py 48 24 --shots 4000 --warm 0 > gpurun_out/ncu_r02h.log 2>&1
