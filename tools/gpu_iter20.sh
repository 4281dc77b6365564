set -x
python -m pytest tests/test_gpu_parity.py -q -x -k fused 2>&1 | tail -2
for f in "--fuse-encode" "" "--fuse-encode"; do timeout 600 python bench.py --no-compare --no-cpu-baseline $f > gpurun_out/b20.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b20.json')); r=d['roofline']
print('$f value',round(d['value'],1),'frac',round(r['frac'],3), 'clk', d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"; done
