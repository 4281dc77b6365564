# configs[3] per GPU (one rank's share of c4 at 8 GPUs): 4096^2 x 512, 8 chunks, k = 4, T = 32
set -x
free -g | head -2
timeout 1800 python bench.py --workload c4slab --steps 3 --warmup 3 --no-compare --no-cpu-baseline > gpurun_out/bench_c4slab.json 2> gpurun_out/bench_c4slab.err
tail -c 1500 gpurun_out/bench_c4slab.err
cat gpurun_out/bench_c4slab.json
