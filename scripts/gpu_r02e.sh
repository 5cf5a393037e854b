# r02e: L2 ceiling + config-4 large-chi forms: rates at k = 13 / 15 / 17 and
# one ncu --set full capture of the block-per-shot wide kernel (n48 t24, k=15)
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/peaks.cu && timeout 120 /tmp/peaks > gpurun_out/peaks_r02e.json 2>&1
for nt in "56 16" "48 24" "40 24" "24 24" "64 24"; do
  timeout 300 python scripts/c4_point.py $nt --shots 20000 >> gpurun_out/c4_r02e.jsonl 2>> gpurun_out/c4_r02e.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 \
  -o gpurun_out/prof_r02e_c4_n48_t24 python scripts/c4_point.py 48 24 --shots 4000 --warm 0 > gpurun_out/ncu_r02e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 \
  -o gpurun_out/prof_r02e_c4_n56_t16 python scripts/c4_point.py 56 16 --shots 8000 --warm 0 >> gpurun_out/ncu_r02e.log 2>&1
