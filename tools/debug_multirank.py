import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth
import paper_2204_11315_b200 as oocs
from paper_2204_11315_b200.dist import LoopbackExchange
R = 4
nx, ny, nz, n, k = 32, 40, 128, 8, 2
vel, p0 = synth.fields(nx, ny, nz)
az = nz + 2 * R
def cfg(store, mode, codec, rank=0, world=1):
    return oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, codec=codec,
                            rate_bits=16, mode=mode, store=store, rank=rank, world=world)
for store, mode, codec in [("host", "swb", "identity"), ("device", "swb", "identity"), ("host", "swb", "blockquant")]:
    for T in (2, 4, 6):
        ref = oocs.Plan(cfg(store, mode, codec))
        for a, arr in enumerate((vel, p0, p0)):
            ref.load(a, arr, 0, az)
        ref.run(T)
        want = [ref.store(a, 0, az) for a in (1, 2)]
        ref.close()
        world = 2
        ex = LoopbackExchange(world)
        plans = []
        for r in range(world):
            pl = oocs.Plan(cfg(store, mode, codec, r, world))
            lo, hi = pl.info.store_lo + R, pl.info.store_hi + R
            for a, arr in enumerate((vel, p0, p0)):
                pl.load(a, np.ascontiguousarray(arr[lo:hi]), lo, hi)
            pl.set_exchange(ex.fn(r))
            plans.append(pl)
        th = [threading.Thread(target=lambda pl=pl: pl.run(T)) for pl in plans]
        [t.start() for t in th]; [t.join() for t in th]
        for pl in plans:
            zl, zh = pl.info.z_lo + R, pl.info.z_hi + R
            lo, hi = pl.info.store_lo + R, pl.info.store_hi + R
            for j, a in enumerate((1, 2)):
                got = pl.store(a, lo, hi)
                d = np.abs(got - want[j][lo:hi]).max(axis=(1, 2))
                bad = [lo + i for i in np.flatnonzero(d > 0)]
                print(store, codec, "T", T, "rank", pl.info.z_lo, "arr", a, "store", (lo, hi), "owned", (zl, zh), "bad planes", bad[:6], "...", bad[-3:] if bad else "")
            pl.close()
