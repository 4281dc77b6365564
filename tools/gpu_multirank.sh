# the N>1 bench contract on one GPU: two ranks sharing cuda:0, halo exchange over gloo (NCCL cannot run
# two ranks on one device); the throughput is not a scaling number, the path is what is exercised
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-compare --no-cpu-baseline > gpurun_out/bench_w2_gloo.json 2> gpurun_out/bench_w2_gloo.err
tail -c 600 gpurun_out/bench_w2_gloo.err
cat gpurun_out/bench_w2_gloo.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_w2_ref.json 2> gpurun_out/bench_w2_ref.err
echo "ref rc=$?"; cat gpurun_out/bench_w2_ref.json
