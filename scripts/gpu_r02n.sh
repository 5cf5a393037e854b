# r02n: config-4 grid on the round-2 build + sanitizers over the new paths
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/config4_sweep.py --shots 50000 --out gpurun_out/config4_sweep_r02n.jsonl > gpurun_out/config4_sweep_r02n.log 2>&1
TAG=r02n bash scripts/gpu_sanitize.sh
