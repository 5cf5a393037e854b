# r02o: large-chi forms at k = 12..15: warp per shot (global chi) vs block per shot
# (16 warps; shared chi / global ping-pong) vs 8-warp blocks (2 per SM)
set -x
mkdir -p gpurun_out
G8=$PWD/paper_2512_23037_b200/variants/libgstab_g8.so
for nt in "20 32" "56 16" "64 16" "48 24" "56 24"; do
  for fl in "" "CHI_BLOCK" "CHI_BLOCK,CHI_GLOBAL"; do
    timeout 300 python scripts/c4_point.py $nt --shots 20000 --flags "$fl" | sed 's/^/g16 /' >> gpurun_out/c4_r02o.txt 2>> gpurun_out/c4_r02o.err
    GSTAB_LIB=$G8 timeout 300 python scripts/c4_point.py $nt --shots 20000 --flags "$fl" | sed 's/^/g8  /' >> gpurun_out/c4_r02o.txt 2>> gpurun_out/c4_r02o.err
  done
done
