set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cp paper_2204_11315_b200/liboocs.so build/liboocs_new.so
bash tools/gpu_ab.sh build/liboocs_base.so build/liboocs_new.so 2
AB_ARGS="--fuse-encode" bash tools/gpu_ab.sh build/liboocs_base.so build/liboocs_new.so 1
