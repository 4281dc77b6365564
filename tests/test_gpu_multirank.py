"""Multi-rank z-slab sharding with the in-library peer-memory halo exchange, on ONE GPU: every rank is its
own process (its own CUDA context, as on an 8-GPU box), plans connected through CUDA IPC handles moved over a
gloo process group (paper_2204_11315_b200.dist.connect).  Edge chunks store their kR encoded planes straight
into the neighbour's ghost slot and signal it with stream memory operations -- the exact code path of a
multi-GPU run, with NVLink replaced by the GPU's own memory.

The sharded result must equal the single-rank run bitwise: each global chunk is computed from identical
inputs whatever GPU owns it.  Split runs must equal one run (run(a); run(b) == run(a+b), including a == k:
the exchange happens after every sweep, the last one included)."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4
NX, NY, NZ, NB, K = 32, 40, 128, 8, 2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _cfg(codec, store, mode, rank=0, world=1, nb=NB, k=K, rate=16):
    dec = store == "device_decv"  # device store with the velocity kept decoded (OOCS_FLAG_DECODED_VELOCITY)
    fuse = store.endswith("_fuse")  # OOCS_FLAG_FUSE_DECODE: interior chunks fused, edge chunks (ghost planes) not
    store = store[:-5] if fuse else store
    return oocs.make_config(nx=NX, ny=NY, nz=NZ, dt=float(synth.dt_for()), n_blocks=nb, tb_depth=k, codec=codec,
                            rate_bits=rate if codec != "identity" else 32, mode=mode,
                            store="device" if dec else store, rank=rank, world=world, decoded_velocity=dec,
                            fuse_decode=fuse)


def _load(pl):
    vel, p0 = synth.fields(NX, NY, NZ)
    lo, hi = pl.info.store_lo + R, pl.info.store_hi + R
    for a, arr in enumerate((vel, p0, p0)):
        pl.load(a, np.ascontiguousarray(arr[lo:hi]), lo, hi)


def _rank_main(rank, world, port, args, steps_list, q):
    """One rank: its own process and CUDA context on cuda:0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OOCS_WATCHDOG_S="120")
    import torch.distributed as dist

    from paper_2204_11315_b200 import dist as odist

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        pl = oocs.Plan(_cfg(*args, rank=rank, world=world))
        _load(pl)
        odist.connect(pl)
        stats = []
        for T in steps_list:
            st = pl.run(T)
            stats.append((st.bytes_h2d, st.bytes_exchange, st.cell_updates))
            dist.barrier()
        zl, zh = pl.info.z_lo + R, pl.info.z_hi + R
        got = {a: pl.read_raw(a, zl, zh) for a in (1, 2)}
        # the ghost planes read back through the slots equal the neighbours' owned planes (checked by the parent)
        sl, sh = pl.info.store_lo + R, pl.info.store_hi + R
        ghosts = {a: pl.read_raw(a, sl, sh) for a in (1, 2)}
        q.put((rank, (zl, zh, sl, sh), got, ghosts, stats, None))
        dist.barrier()
        pl.close()
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        import traceback
        q.put((rank, None, None, None, None, traceback.format_exc()))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded(args, world, steps_list):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, args, steps_list, q)) for r in range(world)]
    [p.start() for p in ps]
    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=300))
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    errs = [r[5] for r in res if r[5]]
    assert not errs, errs[0]
    return sorted(res, key=lambda r: r[0])


def _single(args, T):
    ref = oocs.Plan(_cfg(*args))
    _load(ref)
    ref.run(T)
    az = NZ + 2 * R
    want = {a: ref.read_raw(a, 0, az) for a in (1, 2)}
    pb = ref.info.plane_bytes
    ref.close()
    return want, pb


CASES = [("blockquant", "host", "swb"), ("blockquant", "device", "swb"), ("identity", "host", "dwb"),
         ("blockquant", "device_decv", "swb"), ("zfp", "host", "compress"), ("trunc16", "host", "swb"),
         ("blockquant", "host_fuse", "swb"), ("blockquant", "device_fuse", "swb")]


@pytest.mark.parametrize("args", CASES, ids=lambda a: "-".join(a))
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_equals_single_rank(args, world):
    T = 3 * K
    want, pb = _single(args, T)
    res = _sharded(args, world, [T])
    kR = K * R
    for rank, (zl, zh, sl, sh), got, ghosts, stats, _ in res:
        for a in (1, 2):
            assert np.array_equal(got[a], want[a][zl * pb:zh * pb]), (rank, a)
            # the store's ghost planes mirror the slots the neighbours wrote: S_T of their owned planes
            assert np.array_equal(ghosts[a], want[a][sl * pb:sh * pb]), (rank, a, "ghost")
        h2d, exch, cells = stats[0]
        n_edges = (rank > 0) + (rank + 1 < world)
        assert exch == 3 * n_edges * 2 * kR * pb  # one send per edge per sweep, 2 pressures x kR planes
        assert cells == NX * NY * (zh - zl) * T


@pytest.mark.parametrize("args", [("blockquant", "host", "swb"), ("blockquant", "device", "swb")],
                         ids=lambda a: "-".join(a))
def test_split_runs_equal_one_run(args):
    """after run(a) the neighbours' edge planes of the final state are in the ghost slots,
    so run(a); run(b) == run(a + b) -- also when a == k (a single sweep)."""
    world = 2
    want, pb = _single(args, 4 * K)
    res = _sharded(args, world, [K, K, 2 * K])
    for rank, (zl, zh, *_), got, _g, _s, _ in res:
        for a in (1, 2):
            assert np.array_equal(got[a], want[a][zl * pb:zh * pb]), (rank, a)


def test_host_h2d_skips_ghost_pressure_planes():
    """Out-of-core ranks with neighbours on both sides: their pressure halo never crosses PCIe (only the
    static velocity ghost planes do)."""
    args = ("blockquant", "host", "swb")
    world = 4
    res = _sharded(args, world, [K])
    one = oocs.Plan(_cfg(*args))
    pb = one.info.plane_bytes
    one.close()
    kR = K * R
    for rank, (zl, zh, sl, sh), _g, _gh, stats, _ in res:
        h2d = stats[0][0]
        own = zh - zl
        # per sweep: velocity over the store range, pressures over the owned range plus the physical
        # boundary planes the edge ranks own, nothing more
        lo_b = R if rank == 0 else 0
        hi_b = R if rank == world - 1 else 0
        assert h2d == ((sh - sl) + 2 * (own + lo_b + hi_b)) * pb, (rank, h2d)
        assert sh - sl == own + (kR if rank > 0 else R) + (kR if rank < world - 1 else R)
