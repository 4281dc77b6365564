# same-box A/B: K steps as blocking oocs_run calls vs back-to-back oocs_run_async (value only), alternating
for r in 1 2; do for wl in c3 c4slab; do for mode in sync async; do
  extra=""; [ $mode = sync ] && extra="--sync-steps"
  timeout 900 python bench.py --workload $wl --no-error --no-device-resident --no-compare --no-cpu-baseline $extra > gpurun_out/ab_${wl}_$mode.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_${wl}_$mode.json')); print('$r', '$wl', '$mode', round(d['value'],2), round(d['e2e']['value'],2), d['step_ms_rank0']['all'])"
done; done; done
