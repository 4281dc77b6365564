# Round measurement: GPU tests + smoke, the default bench line, the reference arm, codec variants,
# the ncu launch list of the bench command and ncu --set full of the three hot kernels.
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); e=d['e2e']; r=d['roofline']
print('value',round(d['value'],1),'frac',round(r['frac'],3),'e2e',round(e['value'],2),'pcie',round(e['pcie_frac'],3),'cpu',d['cpu_baseline']['value'],'clk',d['clocks'], {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/bench_ref.json
timeout 600 python bench.py --codec trunc16 --no-compare --no-cpu-baseline > gpurun_out/bench_trunc16.json 2> gpurun_out/bench_trunc16.err
timeout 600 python bench.py --codec zfp --no-compare --no-cpu-baseline > gpurun_out/bench_zfp.json 2> gpurun_out/bench_zfp.err
for f in trunc16 zfp; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); r=d['roofline']
print('$f value',round(d['value'],1),'e2e',round(d['e2e']['value'],2), {k:(round(v['GBps'] or 0),round(v['ms'],1),v['launches']) for k,v in r['per_kernel'].items()})"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bq_|stencil|id_|tr16|zfp" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu-baseline > gpurun_out/launches.log 2>&1
tail -n 2 gpurun_out/launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 12 -c 1 -o gpurun_out/prof_step python tools/profile_kernels.py > gpurun_out/prof_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_decode -s 24 -c 1 -o gpurun_out/prof_dec python tools/profile_kernels.py > gpurun_out/prof_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_encode -s 16 -c 1 -o gpurun_out/prof_enc python tools/profile_kernels.py > gpurun_out/prof_enc.log 2>&1
ls gpurun_out/*.ncu-rep
