set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do for lib in build/liboocs_base.so build/liboocs_v4.so; do
  OOCS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-compare > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']
print('$(basename $lib)','value',round(d['value'],1),'clk',d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),v['launches']) for k,v in r['per_kernel'].items()})"
done; done
