# decode -> first step fusion: bitwise tests, an alternating A/B of the bench (device-resident value and
# per-kernel times), and ncu --set full of one interior c2 chunk with the fusion on
timeout 900 python -m pytest tests/test_gpu_fuse_decode.py -x -q 2>&1 | tail -3
for i in 1 2; do
  for f in "" "--fuse-decode"; do
    timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-error --no-compare $f > gpurun_out/fuse_ab_${i}${f:+_fused}.json 2> gpurun_out/fuse_ab_${i}${f:+_fused}.err
    python - "$f" gpurun_out/fuse_ab_${i}${f:+_fused}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
r = d["value_device_resident"]
pk = d["roofline"]["per_kernel"]
print(sys.argv[1] or "unfused", "ooc", round(d["value"], 2), "resident", round(r["value"], 2), {k: (round(v["ms"], 1), v["launches"]) for k, v in pk.items()}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
  done
done
WL=c2 FUSE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"bq_|stencil" -s 22 -c 7 -o gpurun_out/prof_fuse_c2 python tools/profile_kernels.py > gpurun_out/ncu_fuse.log 2>&1; tail -2 gpurun_out/ncu_fuse.log
