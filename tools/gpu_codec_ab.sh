timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuse_decode.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -3
timeout 1200 python tools/kernel_ab.py build/liboocs_v1.so build/liboocs_codec2.so --rounds 3 2>&1 | tail -6
WL=c2 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"bq_|stencil" -s 18 -c 6 -o gpurun_out/prof_codec2_c2 python tools/profile_kernels.py > gpurun_out/ncu_codec2.log 2>&1; tail -1 gpurun_out/ncu_codec2.log
