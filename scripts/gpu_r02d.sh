# r02d: measured ceilings (issue kernels unrolled), A/B of the T-sweep sign
# masks against HEAD (_ab_base), two warps per shot at k=10 (variant g2), GPU tests
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/peaks.cu && timeout 120 /tmp/peaks > gpurun_out/peaks_r02d.json 2>&1
TAG=r02d_tsign bash scripts/gpu_ab_tree.sh
for so in paper_2512_23037_b200/variants/libgstab_*.so; do
  name=$(basename $so .so)
  GSTAB_LIB=$PWD/$so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_r02d_${name}.json 2>> gpurun_out/ab_r02d_var.err
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02d.log
