"""Representative launches for ncu: one c2 plan with the compressed state in HBM, one warm-up sweep,
then one profiled sweep (8 chunks x [1 decode + k=4 steps + 1 encode] launches for BlockQuant)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402

nx, ny, nz, nb, k, T, rate = bench.WORKLOADS[os.environ.get("WL", "c2")]
codec = sys.argv[sys.argv.index("--codec") + 1] if "--codec" in sys.argv else "blockquant"
if codec == "trunc16":
    rate = 16
# FUSE=1: the decode -> first step fusion (per interior chunk: decode of v and p_t, ring decode of p_{t-1},
# the fused first step, 3 steps, encode)
c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=nb, tb_depth=k, rate_bits=rate,
                     mode="swb", store="device", codec=codec, fuse_decode=os.environ.get("FUSE") == "1")
pl = oocs.Plan(c)
bench.load_state(pl, nx, ny, nz, 0)
pl.run(k)
# the profiled sweep is bracketed by cudaProfilerStart/Stop: run ncu with --profile-from-start off,
# then -s/-c count launches of this sweep only (chunk 3 of 8 is an interior chunk)
import torch  # noqa: E402

torch.cuda.synchronize()
torch.cuda.profiler.start()
st = pl.run(k)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("sweep ms", st.wall_ms, "launches", list(st.kernel_launches))
