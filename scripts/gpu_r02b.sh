set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02b.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/peaks.cu && timeout 120 /tmp/peaks > gpurun_out/peaks_r02b.json 2>&1
timeout 1200 python scripts/msc_rates.py --shots 1e9 > gpurun_out/msc_rates_r02b.jsonl 2> gpurun_out/msc_rates_r02b.err
timeout 600 python bench.py --workload msc_d5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-waves 2 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
timeout 600 python bench.py --workload msc_d3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-waves 2 > gpurun_out/bench_r02b_d3.json 2>> gpurun_out/bench_r02b.err
