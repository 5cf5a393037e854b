# r02g: no-span pivots from the tracked norm + MLP in the block form: tests + config-4 A/B (GS_GUNROLL 4 / 2 / 1)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_reference_semantics.py -q -x > gpurun_out/pytest_r02g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02g.log
for nt in "56 16" "48 24" "40 24" "24 24" "48 32" "20 32"; do
  timeout 300 python scripts/c4_point.py $nt --shots 20000 | sed 's/^/u4 /' >> gpurun_out/c4_r02g.txt 2>> gpurun_out/c4_r02g.err
  for v in u2 u1; do
    GSTAB_LIB=$PWD/paper_2512_23037_b200/variants/libgstab_$v.so timeout 300 python scripts/c4_point.py $nt --shots 20000 | sed "s/^/$v /" >> gpurun_out/c4_r02g.txt 2>> gpurun_out/c4_r02g.err
  done
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
