# r02ee: SplitMix fire-bit ring scanned in bounded steps (long noise stretches inside wide sections): tests + SplitMix A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02ee.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02ee.log
TAG=r02ee_smx bash scripts/gpu_ab_tree.sh --rng splitmix
