# ncu --set full of the fused last-step+encode stencil (mangled name ...Li16ELb1E...) and one plain step
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:Li16ELi1E -s 8 -c 1 -o gpurun_out/prof_fused python tools/profile_kernels.py > gpurun_out/prof_fused.log 2>&1
tail -n 3 gpurun_out/prof_fused.log
