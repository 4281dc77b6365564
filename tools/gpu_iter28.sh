set -x
python -m pytest tests/test_gpu_zfp.py -x -q 2>&1 | tail -2
cp paper_2204_11315_b200/liboocs.so build/liboocs_new.so
AB_ARGS="--codec zfp" bash tools/gpu_ab.sh build/liboocs_zfp2.so build/liboocs_new.so 1
