set -x
python -m pytest tests/test_gpu_zfp.py -x -q 2>&1 | tail -3
cp paper_2204_11315_b200/liboocs.so build/liboocs_new.so
AB_ARGS="--codec zfp" bash tools/gpu_ab.sh build/liboocs_head.so build/liboocs_new.so 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_decode -s 24 -c 1 -o gpurun_out/prof_zfpdec2 python tools/profile_kernels.py --codec zfp > gpurun_out/prof_zfp2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zfp_encode -s 16 -c 1 -o gpurun_out/prof_zfpenc2 python tools/profile_kernels.py --codec zfp >> gpurun_out/prof_zfp2.log 2>&1
tail -n 2 gpurun_out/prof_zfp2.log
