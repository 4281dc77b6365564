# step2 prototype: parity, micro-benchmark, ncu of both variants; codec A/B (old vs new build)
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 600 python -m pytest tests/test_gpu_step2.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python tools/step2_micro.py 2>&1 | tail -4
timeout 600 python tools/kernel_ab.py build/liboocs_old.so build/liboocs_new.so --rounds 2 2>&1 | tail -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_step2_kernel -c 1 -o gpurun_out/prof_step2 python tools/step2_micro.py --seconds 0.2 --out gpurun_out/step2_micro_ncu.json > gpurun_out/ncu_step2.log 2>&1; tail -3 gpurun_out/ncu_step2.log
