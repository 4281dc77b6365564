# ncu --set full of one ZFP decode and one ZFP encode launch (c2, device store)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_decode -s 24 -c 1 -o gpurun_out/prof_zfpdec python tools/profile_kernels.py --codec zfp > gpurun_out/prof_zfp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_encode -s 16 -c 1 -o gpurun_out/prof_zfpenc python tools/profile_kernels.py --codec zfp >> gpurun_out/prof_zfp.log 2>&1
tail -n 3 gpurun_out/prof_zfp.log
