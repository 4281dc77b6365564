timeout 900 ncu --set full --clock-control none --import-source on -k regex:tr16_decode -s 24 -c 1 -o gpurun_out/prof_tr16dec python tools/profile_kernels.py --codec trunc16 > gpurun_out/prof_tr16.log 2>&1
tail -n 2 gpurun_out/prof_tr16.log
