# Truncate-16 codec: GPU parity, c2 bench line with --codec trunc16, accuracy study, full GPU suite
set -x
python -m pytest tests/test_gpu_trunc16.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --codec trunc16 --no-compare > gpurun_out/bench_trunc16.json 2> gpurun_out/bench_trunc16.err
tail -c 600 gpurun_out/bench_trunc16.err
timeout 900 python tools/accuracy.py --codec trunc16 --rates 16 --out gpurun_out/r01_accuracy_trunc16.json > gpurun_out/acc_trunc16.log 2>&1
tail -n 3 gpurun_out/acc_trunc16.log
python -m pytest tests -m gpu -q 2>&1 | tail -3
