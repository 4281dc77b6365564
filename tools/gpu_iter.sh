# quick iteration: GPU tests, c2 bench (x2 for variance), ncu of one stencil + one decode + one encode launch
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-compare > gpurun_out/bench_c2_$i.json 2> gpurun_out/bench_c2_$i.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c2_$i.json')); r=d['roofline']
print('value',round(d['value'],1),'e2e',round(d['e2e']['value'],2),'pcie_frac',round(d['e2e']['pcie_frac'],3),'clk',d['clocks'], {k:round(v['GBps'] or 0) for k,v in r['per_kernel'].items()})"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 12 -c 1 -o gpurun_out/prof_step python tools/profile_kernels.py > gpurun_out/prof_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_decode -s 24 -c 1 -o gpurun_out/prof_dec python tools/profile_kernels.py > gpurun_out/prof_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_encode -s 16 -c 1 -o gpurun_out/prof_enc python tools/profile_kernels.py > gpurun_out/prof_enc.log 2>&1
tail -3 gpurun_out/prof_step.log
