# lanes 2 vs 3 on every out-of-core workload (value only)
for wl in c3 c2 c4slab beyond_hbm; do for l in 3 2; do
  timeout 900 python bench.py --workload $wl --lanes $l --steps 3 --warmup 2 --no-error --no-device-resident --no-compare --no-cpu-baseline > gpurun_out/lanes_${wl}_$l.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lanes_${wl}_$l.json')); print('$wl', $l, round(d['value'],2), round(d['roofline_pcie']['frac_of_bound_5050'],3), d['peak_gpu_mem_gb'])"
done; done
