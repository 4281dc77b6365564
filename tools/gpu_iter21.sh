set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b21.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b21.json')); r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2), d['compare'])"
