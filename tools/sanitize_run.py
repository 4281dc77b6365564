"""Small runs of every hot-path kernel and schedule for compute-sanitizer (memcheck / racecheck /
synccheck): ragged grids, every codec, host and device stores, Alg. 1 and DAG schedules, the resident
(compressed / decoded) velocity flags, both stencils, the BASELINE mode (its carry is an SM copy too)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402

R = 4
nx, ny, nz = 44, 36, 48
vel, p0 = synth.fields(nx, ny, nz)
az = nz + 2 * R
for codec, rate in (("blockquant", 16), ("blockquant", 24), ("zfp", 12), ("trunc16", 16), ("identity", 32)):
    for store, sched, mode, extra in (("host", "alg1", "swb", {}), ("device", "alg1", "swb", {}),
                                      ("host", "dag_func", "dwb", {}),
                                      ("device", "alg1", "swb", {"decoded_velocity": True}),
                                      ("host", "alg1", "swb", {"resident_velocity": True}),
                                      ("host", "alg1", "compress", {"stencil": "star7"}),
                                      ("host", "alg1", "baseline", {}) if codec == "identity" else
                                      ("device", "alg1", "dwb", {"stencil": "star7"})):
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=3, tb_depth=2, codec=codec,
                             rate_bits=rate, mode=mode, store=store, schedule=sched, **extra)
        pl = oocs.Plan(c)
        for a, arr in enumerate((vel, p0, p0)):
            pl.load(a, arr, 0, az)
        pl.run(4)
        out = pl.store(2, 0, az)
        assert np.isfinite(out).all()
        pl.close()
        print("ok", codec, rate, store, sched, mode, extra, flush=True)
# chained runs (oocs_run_async): a run issued while the previous one drains
c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=3, tb_depth=2, codec="blockquant",
                     rate_bits=16, mode="swb", store="host", n_lanes=2)
pl = oocs.Plan(c)
for a, arr in enumerate((vel, p0, p0)):
    pl.load(a, arr, 0, az)
for _ in range(3):
    pl.run_async(2)
assert len(pl.wait()) == 3
assert np.isfinite(pl.store(2, 0, az)).all()
pl.close()
print("ok chained", flush=True)
