"""Experiment: per-step error of the GPU stencil vs the fp64 oracle (max|g-o|/max|o|) on paper-like fields,
for whichever liboocs is loaded (OOCS_LIB).  Prints the max over several grids and states."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, oracle, synth
import paper_2204_11315_b200 as oocs
from test_gpu_parity import to_ws, from_ws, stream
R = 4
worst = 0
for (nx, ny, nz) in [(64, 64, 64), (128, 96, 40), (256, 256, 24)]:
    vel, p0 = synth.fields(nx, ny, nz)
    dt = synth.dt_for()
    pp, pc = oracle.incore(vel, p0.copy(), p0.copy(), dt, 7)  # an evolved state
    az, ay, ax = pc.shape
    o = pp.copy()
    oracle.step(vel, o, pc, dt, R, az - R)
    tv, tp, tc = to_ws(vel), to_ws(pp), to_ws(pc)
    oocs.oocs_step(tv.data_ptr(), tp.data_ptr(), tc.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R, stream())
    torch.cuda.synchronize()
    g = from_ws(tp, ax)
    sl = (slice(R, az - R), slice(R, ay - R), slice(R, ax - R))
    e = np.max(np.abs(g[sl].astype(np.float64) - o[sl])) / np.max(np.abs(o[sl]))
    ulp = np.max(np.abs(g[sl].view(np.int32).astype(np.int64) - o[sl].view(np.int32).astype(np.int64)))
    worst = max(worst, e)
    print(os.environ.get("OOCS_LIB", "default"), (nx, ny, nz), "max rel err", e, "max ulp diff", ulp)
print("WORST", worst)
