# round-end style check: all GPU tests, smoke, the default bench line, the reference arm
python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); e=d['e2e']
print('value',round(d['value'],1),'frac',round(d['roofline']['frac'],3),'e2e',round(e['value'],2),'pcie',round(e['pcie_frac'],3),'cpu',d['cpu_baseline']['value'],'clk',d['clocks'])"
