set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for f in "" "--single-stream-lanes"; do timeout 600 python tools/timeline.py $f --out gpurun_out/tl$f.json > gpurun_out/tl$f.log 2>&1; grep -E "wall_ms|gcell|\"H2D\"" gpurun_out/tl$f.log; tail -n 4 gpurun_out/tl$f.log; done
timeout 600 python bench.py --no-compare --no-cpu-baseline > gpurun_out/b10.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b10.json')); e=d['e2e']; print('value',round(d['value'],1),'e2e',round(e['value'],2), 'pcie_frac', e.get('pcie_frac'), {k:v for k,v in e.items() if 'resident' in k})"
