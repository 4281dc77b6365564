# fused last step + encode: parity, then bench with and without fusion
set -x
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for f in "" "--no-fusion" ""; do timeout 600 python bench.py --no-cpu-baseline --no-compare $f > gpurun_out/b5.json 2> gpurun_out/b5.err; python -c "
import json; d=json.load(open('gpurun_out/b5.json')); r=d['roofline']
print('$f value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2),'clk',d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"; done
