# lanes 2 / 3 / 4 on the final pipeline: c3 out-of-core timeline (throughput, busy fractions) and arena
for l in 2 3 4; do
  timeout 600 python tools/timeline.py --workload c3 --lanes $l --out gpurun_out/timeline_c3_lanes$l.json 2>&1 | grep -E "gcell|h2d_while|tail_ms" | head -3
done
python -c "
import paper_2204_11315_b200 as o, synth
for l in (2,3,4):
    c=o.make_config(nx=2048,ny=2048,nz=2048,dt=float(synth.dt_for()),n_blocks=16,tb_depth=4,mode='swb',store='host',n_lanes=l)
    print(l, o.oocs_plan_estimate(c).arena_bytes/1e9)
c=o.make_config(nx=2048,ny=2048,nz=2048,dt=float(synth.dt_for()),n_blocks=16,tb_depth=4,mode='baseline',codec='identity',rate_bits=32,store='host')
print('baseline', o.oocs_plan_estimate(c).arena_bytes/1e9)
"
