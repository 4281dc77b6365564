# end-of-round check on the final code: the -m gpu suite, compute-sanitizer, and the bench line
export OOCS_REPORT_DIR=gpurun_out/rep
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitizer/sanitize_$tool.log | head -3
done
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
