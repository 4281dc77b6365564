# the pipeline schedule after a change: the whole -m gpu suite (incl. full-size two-sweep parity), the c3
# timeline and the bench line
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/timeline.py --workload c3 --out gpurun_out/timeline_c3_r02.json 2>&1 | grep -E "gcell|h2d_while|tail_ms" | head -4
timeout 900 python bench.py > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; python -c "
import json; d=json.load(open('gpurun_out/bench_pipe.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'pcie frac', d['roofline_pcie']['frac_of_bound'], d['roofline_pcie']['frac_of_bound_5050'], 'dev', d['value_device_resident']['value'], 'stencil', d['roofline']['frac'])"
