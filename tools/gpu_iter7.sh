# trunc16 kernels v2 + timeline: tests, trunc16 bench line, c2 timelines (host store, resident velocity)
set -x
python -m pytest tests/test_gpu_trunc16.py tests/test_gpu_timeline.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --codec trunc16 --no-compare --no-cpu-baseline > gpurun_out/bench_trunc16b.json 2> gpurun_out/bench_trunc16b.err
python -c "
import json; d=json.load(open('gpurun_out/bench_trunc16b.json')); r=d['roofline']
print('value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"
timeout 600 python tools/timeline.py --out gpurun_out/r01_timeline_c2.json > gpurun_out/timeline.log 2>&1
timeout 600 python tools/timeline.py --resident-velocity --out gpurun_out/r01_timeline_c2_resv.json > gpurun_out/timeline_resv.log 2>&1
cat gpurun_out/timeline.log
tail -n 8 gpurun_out/timeline_resv.log
