# end-of-round check on the final code: the -m gpu suite (with the full-size parity reports) and the bench
# line.  compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset), so the
# sanitizer pass (tools/gpu_sanitize.sh, tools/sanitize_run.py) is no longer part of it.
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
