# H2D issued before the carry (and the carry as an SM copy): timeline and bench on c3, pipeline parity
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize_c3.py 2>&1 | tail -3
timeout 600 python tools/timeline.py --workload c3 --out gpurun_out/timeline_c3_r02.json 2>&1 | grep -E "gcell|h2d_while|tail_ms" | head -4
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; python -c "
import json; d=json.load(open('gpurun_out/bench_pipe.json')); print('value', d['value'], 'pcie frac', d['roofline_pcie']['frac_of_bound'], d['roofline_pcie']['frac_of_bound_5050'], 'dev', d['value_device_resident']['value'])"
