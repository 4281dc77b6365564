set -x
python -m pytest tests/test_gpu_trunc16.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --codec trunc16 --no-compare --no-cpu-baseline > gpurun_out/bench_trunc16.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_trunc16.json')); r=d['roofline']
print('value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"
