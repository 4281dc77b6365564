# end-of-round measurement refresh: GPU tests, smoke, bench line (+ codec variants), reference arm,
# ncu launch list of the bench command, ncu --set full of one interior-chunk stencil / decode / encode
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 1500 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in zfp trunc16; do timeout 600 python bench.py --codec $c --no-compare --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bq_|stencil|id_" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu-baseline > gpurun_out/launches.log 2>&1
tail -2 gpurun_out/launches.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stencil_step -s 12 -c 1 -o gpurun_out/prof_step python tools/profile_kernels.py > gpurun_out/prof_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bq_decode -s 3 -c 1 -o gpurun_out/prof_dec python tools/profile_kernels.py > gpurun_out/prof_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bq_encode -s 3 -c 1 -o gpurun_out/prof_enc python tools/profile_kernels.py > gpurun_out/prof_enc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stencil_step -s 15 -c 1 -o gpurun_out/prof_fused python tools/profile_kernels.py --fuse > gpurun_out/prof_fused.log 2>&1
tail -2 gpurun_out/prof_enc.log gpurun_out/prof_fused.log
ls gpurun_out
