#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (one gpurun call):
#   TAG=x bash scripts/gpu_sanitize.sh   -> gpurun_out/sanitize_TAG.txt
mkdir -p gpurun_out
TAG=${TAG:-x}
OUT=gpurun_out/sanitize_${TAG}.txt
CS="compute-sanitizer --print-limit 20"
{
echo "## memcheck: storage variants (warp / block per shot, smem / global chi, ping-pong block form, narrow limit 5, sparse form), shot indices > 2^32, large-chi block form, cancelled-T span at k=22 (sparse), the sparse-form tests"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_sparse.py -q -m gpu -k "storage or beyond_32 or large_chi or cancelled or sparse" 2>&1 | tail -4
echo "## racecheck: block-per-shot form (shared chi + group scratch), warp form"
timeout 1200 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "storage_modes_match_oracle and (chi_block or default or narrow_k5)" 2>&1 | tail -4
echo "## synccheck: block-per-shot form"
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "chi_block or large_chi" 2>&1 | tail -4
} > $OUT 2>&1
cat $OUT
