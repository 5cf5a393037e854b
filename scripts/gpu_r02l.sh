# r02l: narrow kernel templated on the narrow limit (kn=5 build at 3 blocks,
# 8 queue loads in flight): A/B vs HEAD cc046d9, parity subset
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "golden or storage_modes or oracle" > gpurun_out/pytest_r02l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02l.log
TAG=r02l bash scripts/gpu_ab_tree.sh
