"""Does per-launch event timing (OOCS_FLAG_PROFILE) cost throughput on the value path?  c2, device store."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402

nx, ny, nz, nb, k, T, rate = bench.WORKLOADS["c2"]
dt = float(synth.dt_for())
res = {}
base = None
for prof in (True, False, True, False):
    pl = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nb, tb_depth=k, rate_bits=rate, mode="swb",
                                    store="device", profile=prof))
    if base is None:
        bench.load_state(pl, nx, ny, nz, 0)
        base = pl
        keep = pl
    else:
        bench.copy_state(keep, pl)
    for _ in range(3):
        pl.run(T)
    ms = [pl.run(T).wall_ms for _ in range(4)]
    print("profile" if prof else "no-profile", [round(m, 2) for m in ms], "Gcu/s", round(nx * ny * nz * T / (min(ms) * 1e-3) / 1e9, 1))
    if pl is not keep:
        pl.close()
