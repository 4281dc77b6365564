# A/B of two liboocs builds on the same box: bench.py (no cpu baseline / compare), alternating
# usage: bash tools/gpu_ab.sh OLD.so NEW.so [rounds]   (extra bench args in $AB_ARGS)
A=$1; B=$2; N=${3:-2}
for i in $(seq 1 $N); do for lib in $A $B; do
  OOCS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-compare $AB_ARGS > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']
print('$(basename $lib)','value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],2),'clk',d['clocks']['sm_mhz'], {k:(round(v['GBps'] or 0),v['launches']) for k,v in r['per_kernel'].items()})"
done; done
