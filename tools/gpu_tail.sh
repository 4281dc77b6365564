# chained runs: the run tail's D2Hs issued behind device-side waits (t1) vs host-polled (t0): same box,
# alternating; plus the chained-run bitwise tests with the tail on
true
for r in 1 2 3 4; do
  for L in t0 t1; do
    OOCS_LIB=build/liboocs_$L.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-error --no-compare --no-device-resident > gpurun_out/tail_${L}_${r}.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/tail_${L}_${r}.json').read().strip().splitlines()[-1])
print('$L', round(d['value'],3), round(d['e2e']['value'],3), d['step_ms_rank0']['all'] if 'step_ms_rank0' in d else '')"
  done
done
