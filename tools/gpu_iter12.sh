set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for ex in dispatch single split; do
  timeout 600 python tools/timeline.py --executor $ex --out gpurun_out/tl_$ex.json > gpurun_out/tl_$ex.log 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl_$ex.json')); print('$ex', round(d['gcell_updates_per_s'],2), 'h2d_busy', round(d['busy_frac']['H2D'],3), 'gaps', len(d['h2d_gaps']), 'h2d_gbs', round(d['h2d_while_busy_gbs'],1), 'tail', round(d['h2d_tail_ms'],1), 'enq', round(d['host_enqueue_ms'],1))"
done
tail -n 4 gpurun_out/tl_dispatch.log
timeout 600 python bench.py --no-compare --no-cpu-baseline > gpurun_out/b12.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b12.json')); e=d['e2e']; print('value',round(d['value'],1),'e2e',round(e['value'],2), 'pcie_frac', e.get('pcie_frac'), e.get('resident_velocity_variant',{}).get('value'))"
