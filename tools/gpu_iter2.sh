set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 1500 gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); e=d['e2e']
print('value',round(d['value'],1),'frac',round(d['roofline']['frac'],3),'e2e',round(e['value'],2),'pcie_frac',round(e['pcie_frac'],3),'5050',round(e['pcie_frac_5050'],3),'resident_v',e['resident_velocity_variant'],'clk',d['clocks'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload c1 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err
cat gpurun_out/bench_gloo2.json; tail -5 gpurun_out/bench_gloo2.err
