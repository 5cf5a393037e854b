# r02s: narrow k-split (the k<=4 stretch before the first 2^5-row op keeps the 20-warp layout): A/B vs c434bc9 + parity subset
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "golden or storage_modes or oracle or chunking or lane_per_shot" > gpurun_out/pytest_r02s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02s.log
TAG=r02s bash scripts/gpu_ab_tree.sh
