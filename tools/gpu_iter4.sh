set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for s in alg1 dag dag_func; do timeout 900 python bench.py --no-cpu-baseline --no-compare --schedule $s > gpurun_out/bench_$s.json 2> gpurun_out/bench_$s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$s.json')); e=d['e2e']
print('$s','value',round(d['value'],1),'e2e',round(e['value'],2),'pcie_frac',round(e['pcie_frac'],3),'resv',round(e['resident_velocity_variant']['value'],2))"; done
