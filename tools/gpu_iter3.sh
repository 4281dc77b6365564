set -x
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 2400 python tools/sweep.py > gpurun_out/sweep.log 2>&1
tail -20 gpurun_out/sweep.log
cp profiles/r01_sweep_c3.json gpurun_out/ 2>/dev/null
