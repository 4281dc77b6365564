"""Multi-rank z-slab sharding on ONE GPU: every rank is its own plan (rank r of world W) driven from its
own host thread, halos exchanged through the in-process loopback behind the same callback interface
NCCL uses (paper_2204_11315_b200.dist).  The sharded result must equal the single-rank run bitwise:
each global chunk is computed from identical inputs whatever GPU owns it."""
import threading

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from paper_2204_11315_b200.dist import LoopbackExchange  # noqa: E402

R = 4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _cfg(nx, ny, nz, n, k, codec, store, mode, rank=0, world=1):
    dec = store == "device_decv"  # device store with the velocity kept decoded (OOCS_FLAG_DECODED_VELOCITY)
    return oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, codec=codec,
                            rate_bits=16, mode=mode, store="device" if dec else store, rank=rank, world=world,
                            decoded_velocity=dec)


@pytest.mark.parametrize("store,mode,codec", [("host", "swb", "blockquant"), ("device", "swb", "blockquant"),
                                              ("host", "baseline", "identity"), ("host", "dwb", "identity"),
                                              ("device_decv", "swb", "blockquant")])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_equals_single_rank(store, mode, codec, world):
    nx, ny, nz, n, k, T = 32, 40, 128, 8, 2, 6
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    ref = oocs.Plan(_cfg(nx, ny, nz, n, k, codec, store, mode))
    for a, arr in enumerate((vel, p0, p0)):
        ref.load(a, arr, 0, az)
    ref.run(T)
    want = [ref.read_raw(a, 0, az) for a in (1, 2)]
    pb = ref.info.plane_bytes
    ref.close()

    ex = LoopbackExchange(world)
    plans = []
    for r in range(world):
        pl = oocs.Plan(_cfg(nx, ny, nz, n, k, codec, store, mode, r, world))
        lo, hi = pl.info.store_lo + R, pl.info.store_hi + R
        for a, arr in enumerate((vel, p0, p0)):
            pl.load(a, np.ascontiguousarray(arr[lo:hi]), lo, hi)
        pl.set_exchange(ex.fn(r))
        plans.append(pl)
    errs = []

    def go(pl):
        try:
            st = pl.run(T)
            if world > 1:
                assert st.bytes_exchange > 0
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=go, args=(pl,)) for pl in plans]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    assert not errs, errs
    for pl in plans:
        zl, zh = pl.info.z_lo + R, pl.info.z_hi + R
        for j, a in enumerate((1, 2)):
            got = pl.read_raw(a, zl, zh)
            assert np.array_equal(got, want[j][zl * pb:zh * pb]), (pl.info.z_lo, a)
        pl.close()
