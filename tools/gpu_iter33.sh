set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-compare --no-cpu-baseline > gpurun_out/b33.json 2> gpurun_out/b33.err
tail -c 1000 gpurun_out/b33.err
python -c "
import json; d=json.load(open('gpurun_out/b33.json')); r=d['roofline']
print('value',round(d['value'],1),'dv',d['value_decoded_velocity_variant'],'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2),'clk',d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),v['launches']) for k,v in r['per_kernel'].items()})"
