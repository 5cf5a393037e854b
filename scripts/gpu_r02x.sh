# r02x: large-sample statistical parity (GPU Philox vs CPU oracle SplitMix) on the Table-2 workloads and the others
set -x
mkdir -p gpurun_out
GS_LONG_STATS=1 timeout 2400 python -m pytest tests/test_gpu_statistics_long.py -m gpu -s -q > gpurun_out/long_stats_r02x.log 2>&1
echo "rc=$?" >> gpurun_out/long_stats_r02x.log
