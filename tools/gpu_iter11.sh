# copy chunking x lane stream mapping, c2 host-store timeline
set -x
python -m pytest tests/test_gpu_timeline.py tests/test_gpu_parity.py -q -x -k "timeline or lossy_modes or identity_pipeline" 2>&1 | tail -2
for c in 0 2 8 32; do for f in "" "--single-stream-lanes"; do
  OOCS_COPY_CHUNK_MB=$c timeout 600 python tools/timeline.py $f --out gpurun_out/tl_c$c$f.json > gpurun_out/tl_c$c$f.log 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl_c$c$f.json')); print('chunk $c $f', round(d['gcell_updates_per_s'],2), 'h2d_busy', round(d['busy_frac']['H2D'],3), 'gaps', len(d['h2d_gaps']), 'h2d_gbs', round(d['h2d_while_busy_gbs'],1), 'enq', round(d['host_enqueue_ms'],1))"
done; done
