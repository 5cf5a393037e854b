# r02u: paper Fig. 3 / Fig. 4 analogues through the CLI on the Table-2 d=5 circuit
set -x
mkdir -p gpurun_out
python -m paper_2512_23037_b200 msc --d 5 --out /tmp/msc_d5.stim
python -m paper_2512_23037_b200 msc --d 5 --noise 0.001 --out /tmp/msc_d5_p1e-3.stim
# Fig. 4: throughput vs shots resident per launch (batch_size), p = 1e-3
timeout 900 python -m paper_2512_23037_b200 bench /tmp/msc_d5_p1e-3.stim --sweep batch-size \
  --values 1024,4096,16384,65536,262144,1048576,4194304,16777216 --shots 33554432 --postselect --rng philox \
  --out gpurun_out/fig4_batch_size_r02u.csv
# Fig. 3: throughput vs noise strength (post-selection), 2^25 shots per point
timeout 900 python -m paper_2512_23037_b200 bench /tmp/msc_d5.stim --sweep noise \
  --values 0.0001,0.0002,0.0005,0.001,0.002,0.003,0.005 --shots 33554432 --postselect --rng philox \
  --out gpurun_out/fig3_noise_r02u.csv
cat gpurun_out/fig4_batch_size_r02u.csv gpurun_out/fig3_noise_r02u.csv
