set -x
WL=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_decode -s 24 -c 1 -o gpurun_out/prof_zdec python tools/profile_kernels.py --codec zfp > gpurun_out/prof_zdec.log 2>&1
WL=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_encode -s 16 -c 1 -o gpurun_out/prof_zenc python tools/profile_kernels.py --codec zfp > gpurun_out/prof_zenc.log 2>&1
tail -n 3 gpurun_out/prof_zdec.log
