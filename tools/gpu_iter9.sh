set -x
for c in 8 32; do CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 python tools/timeline.py --out gpurun_out/tl_conn$c.json > gpurun_out/tl_conn$c.log 2>&1; grep -E "wall_ms|gcell" gpurun_out/tl_conn$c.log; done
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python bench.py --no-compare --no-cpu-baseline > gpurun_out/b_conn32.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b_conn32.json')); print('conn32 value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), d['e2e'].get('resident_velocity'))"
