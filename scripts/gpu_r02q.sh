# r02q: 8-warp block form at k = 13-14 (auto): parity + config-4 points
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_r02q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02q.log
for nt in "20 32" "56 16" "64 16" "48 24" "56 24" "40 24" "24 24"; do
  timeout 300 python scripts/c4_point.py $nt --shots 20000 >> gpurun_out/c4_r02q.txt 2>> gpurun_out/c4_r02q.err
done
