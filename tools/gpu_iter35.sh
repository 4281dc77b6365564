set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
cp paper_2204_11315_b200/liboocs.so build/liboocs_new.so
for i in 1 2; do for lib in build/liboocs_base.so build/liboocs_new.so; do for fz in "" "--fuse-encode"; do
  OOCS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-compare --steps 3 $fz > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']
print('$(basename $lib) $fz','value',round(d['value'],1),'dv',round(d['value_decoded_velocity_variant']['value'],1),'clk',d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),v['launches']) for k,v in r['per_kernel'].items()})"
done; done; done
