# full bench line + ncu launch list of the bench command (our kernels only)
set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/bench_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bq_|stencil|id_" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-compare --no-cpu-baseline > gpurun_out/launches.log 2>&1
tail -2 gpurun_out/launches.log
