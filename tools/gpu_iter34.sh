set -x
bash tools/gpu_sanitize.sh
ls gpurun_out
