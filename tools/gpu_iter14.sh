set -x
python -m pytest tests/test_gpu_zfp.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --codec zfp --no-compare --no-cpu-baseline > gpurun_out/bench_zfp2.json 2> gpurun_out/bench_zfp2.err
timeout 600 python bench.py --no-compare --no-cpu-baseline > gpurun_out/bench_bq2.json 2> gpurun_out/bench_bq2.err
for f in zfp2 bq2; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); r=d['roofline']
print('$f value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"; done
