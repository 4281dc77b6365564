set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
cp paper_2204_11315_b200/liboocs.so build/liboocs_new.so
bash tools/gpu_ab.sh build/liboocs_head.so build/liboocs_new.so 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bq_ -s 40 -c 2 -o gpurun_out/prof_codec2 python tools/profile_kernels.py > gpurun_out/prof_codec2.log 2>&1
tail -2 gpurun_out/prof_codec2.log
