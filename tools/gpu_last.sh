# last check of the round: GPU tests, smoke, default bench line (+ reference arm)
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 600 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); e=d['e2e']; r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'dv',d['value_decoded_velocity_variant'].get('value'),'e2e',round(e['value'],2),'pcie',round(e['pcie_frac'],3),'clk',d['clocks'])"
