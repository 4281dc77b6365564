# re-entry check: all GPU tests, smoke, default bench line
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); e=d['e2e']; r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(e['value'],2),'pcie',round(e['pcie_frac'],3),'clk',d['clocks'], {k:round(v['GBps'] or 0) for k,v in r['per_kernel'].items()})"
