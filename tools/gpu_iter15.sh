set -x
python -m pytest tests/test_gpu_zfp.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -4
timeout 600 python bench.py --codec zfp --no-compare --no-cpu-baseline > gpurun_out/bench_zfp3.json 2> gpurun_out/bench_zfp3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_zfp3.json')); r=d['roofline']
print('zfp value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"
