# PCIe-side experiments: link sharing under paced D2H, c3 pipeline timelines with 3 and 4 lanes, the box
# measurement (multi-threaded host copy bandwidth), and the reference arm.
timeout 300 python tools/pcie_pacing.py 2>&1 | tail -10
timeout 600 python tools/timeline.py --workload c3 --out gpurun_out/timeline_c3_l3.json 2>&1 | grep -E "gcell|busy_frac|h2d_while|d2h_while|head|tail|H2D \|" -A0 | head -12
timeout 600 python tools/timeline.py --workload c3 --lanes 4 --out gpurun_out/timeline_c3_l4.json 2>&1 | grep -E "gcell|h2d_while|head_ms|tail_ms" | head -6
timeout 300 python tools/measure_box.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/measure_box.json')); print(d['host_memcpy_gbs_by_threads'], d['numa_nodes'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
