set -x
timeout 600 python tools/timeline.py --out gpurun_out/tl_dispatch.json > gpurun_out/tl_dispatch.log 2>&1
tail -n 12 gpurun_out/tl_dispatch.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_w2_ref.json 2> gpurun_out/bench_w2_ref.err
cat gpurun_out/bench_w2_ref.json | cut -c1-200; grep -o '"cpu_baseline": {[^}]*}' gpurun_out/bench_w2_ref.json
