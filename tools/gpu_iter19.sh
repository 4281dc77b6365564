set -x
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-compare --no-cpu-baseline > gpurun_out/b19.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b19.json')); r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2), 'clk', d['clocks'], {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"
