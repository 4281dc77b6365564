# the other bench workloads on the final code: configs[3]'s per-GPU slab, the beyond-HBM grid, and the
# 2-rank torchrun contract over the IPC exchange on one GPU
timeout 900 python bench.py --workload c4slab --no-compare --no-cpu-baseline > gpurun_out/bench_c4slab.json 2> gpurun_out/bench_c4slab.err; tail -c 200 gpurun_out/bench_c4slab.json
timeout 900 python bench.py --workload beyond_hbm --no-compare --no-cpu-baseline --no-error --no-device-resident --steps 3 --warmup 3 > gpurun_out/bench_beyond.json 2> gpurun_out/bench_beyond.err; tail -c 200 gpurun_out/bench_beyond.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload c2 --dist-backend gloo --steps 3 --warmup 3 > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err; tail -c 300 gpurun_out/bench_w2.json
