set -x
python tools/measure_box.py > gpurun_out/measure_box.log 2>&1
python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -c 3000 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_kernels.py > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 12 -c 1 -o gpurun_out/prof_step python tools/profile_kernels.py > gpurun_out/prof_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_ -s 40 -c 2 -o gpurun_out/prof_codec python tools/profile_kernels.py > gpurun_out/prof_codec.log 2>&1
ls -la gpurun_out
