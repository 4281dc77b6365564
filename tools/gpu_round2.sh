# Round-2 GPU pass: the -m gpu suite (incl. the full-size c3 / c4slab parity), a same-box A/B of the codec
# kernels (build/liboocs_old.so = the round-1 encoder/decoder), ncu --set full of one interior c2 chunk
# (decode, 4 steps, encode), the ncu launch list of the bench command, and the bench line itself.
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6
[ -f build/liboocs_old.so ] && timeout 900 python tools/kernel_ab.py build/liboocs_old.so build/liboocs_new.so --rounds 3 2>&1 | tail -8
WL=c2 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"bq_|stencil" -s 18 -c 6 -o gpurun_out/prof_r02_c2 python tools/profile_kernels.py > gpurun_out/ncu_r02.log 2>&1; tail -2 gpurun_out/ncu_r02.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -c 300 gpurun_out/bench_under_ncu.log
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -c 400 gpurun_out/bench_r02.json
