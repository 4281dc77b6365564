# codec launches batched over arrays: GPU tests + 2 bench runs
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-compare > gpurun_out/bench_c2_$i.json 2> gpurun_out/bench_c2_$i.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c2_$i.json')); r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2),'launches',d['gpu_launches'],'clk',d['clocks'], {k:(round(v['GBps'] or 0),v['launches']) for k,v in r['per_kernel'].items()})"; done
