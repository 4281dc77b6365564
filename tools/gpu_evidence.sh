# launch list of the bench command as it now runs (K steps chained with oocs_run_async), the reference
# arm, and a second bench line on the same box
set -x
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 300 gpurun_out/bench_reference.json
timeout 900 python bench.py > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; tail -c 200 gpurun_out/bench_a.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-error --no-device-resident --no-compare \
  > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"; tail -c 300 gpurun_out/ncu_bench.log
