# BASELINE configs[2] k x rate sweep on the final code
set -x
timeout 3300 python tools/sweep.py --out gpurun_out/sweep_c3.json > gpurun_out/sweep_c3.log 2>&1
tail -5 gpurun_out/sweep_c3.log
