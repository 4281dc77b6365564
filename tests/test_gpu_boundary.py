"""GPU tests of the ABI-2 boundary items: the STAR7 stencil (R = 1, small exact tests),
the CFL check of a loaded velocity, and caller-owned streams (oocs_config.ext_streams).

STAR7: one GPU step against the oracle's (fp64) within the 1e-6 normwise bar; the Identity out-of-core
pipeline bitwise equal to the GPU's own in-core STAR7 run (temporal-blocking validity) and within
the per-step tolerance of the oracle's in-core run; the BlockQuant pipeline against the oracle pipeline
(within one quantisation step per sweep, as the 25-point tests).  Grids span several CTA tiles and a
ragged tail."""
import time

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from test_gpu_parity import _rel_err, from_ws, load_fields, stream, to_ws  # noqa: E402

R = 4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def _plan(nx, ny, nz, n, k, codec="identity", rate=16, **kw):
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, codec=codec,
                         rate_bits=rate, mode="swb", **kw)
    return oocs.Plan(c)


@pytest.mark.parametrize("shape", [(100, 36, 40), (64, 16, 12)])
def test_star7_step_vs_oracle(shape):
    nx, ny, nz = shape
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(3)
    pprev = np.ascontiguousarray(p0 * np.float32(0.9) + rng.normal(scale=1e-3, size=p0.shape).astype(np.float32))
    dt = synth.dt_for()
    az, ay, ax = p0.shape
    o = pprev.copy()
    oracle.step(vel, o, p0, dt, R, az - R, stencil=oracle.STENCIL_STAR7)
    tv, tp, tc = to_ws(vel), to_ws(pprev), to_ws(p0)
    oocs.oocs_step(tv.data_ptr(), tp.data_ptr(), tc.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                   stream(), stencil="star7")
    torch.cuda.synchronize()
    g = from_ws(tp, ax)
    sl = (slice(R, az - R), slice(R, ay - R), slice(R, ax - R))
    assert _rel_err(g[sl], o[sl].astype(np.float64)) <= 1e-6
    # halo untouched, and not the 25-point result
    assert np.array_equal(g[:R], pprev[:R]) and np.array_equal(g[:, :, :R], pprev[:, :, :R])
    o25 = pprev.copy()
    oracle.step(vel, o25, p0, dt, R, az - R)
    assert _rel_err(g[sl], o25[sl].astype(np.float64)) > 1e-4


@pytest.mark.parametrize("n,k,store", [(4, 2, "host"), (3, 1, "host"), (2, 3, "device")])
def test_star7_identity_pipeline_bitwise_equals_gpu_incore(n, k, store):
    nx, ny, nz = 68, 20, 72
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = p0.shape
    T = 2 * k
    dt = synth.dt_for()
    pl = _plan(nx, ny, nz, n, k, store=store, stencil="star7")
    load_fields(pl, vel, p0)
    st = pl.run(T)
    assert st.cell_updates == nx * ny * nz * T
    got_p, got_c = pl.store(1, 0, az), pl.store(2, 0, az)
    pl.close()
    # the GPU's own in-core STAR7 run (oocs_step over the whole grid)
    tv, ta, tb = to_ws(vel), to_ws(p0), to_ws(p0)
    for _ in range(T):
        oocs.oocs_step(tv.data_ptr(), ta.data_ptr(), tb.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                       stream(), stencil="star7")
        ta, tb = tb, ta
    torch.cuda.synchronize()
    assert np.array_equal(got_p.view(np.uint32), from_ws(ta, ax).view(np.uint32))
    assert np.array_equal(got_c.view(np.uint32), from_ws(tb, ax).view(np.uint32))
    _, oc = oracle.incore(vel, p0.copy(), p0.copy(), dt, T, stencil=oracle.STENCIL_STAR7)
    sl = (slice(R, az - R), slice(R, ay - R), slice(R, ax - R))
    assert _rel_err(got_c[sl], oc[sl].astype(np.float64)) <= T * 1e-6


def test_star7_blockquant_pipeline_vs_oracle_pipeline():
    nx, ny, nz, n, k, rate = 68, 20, 72, 3, 2, 16
    q = rate - 1
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = p0.shape
    dt = synth.dt_for()
    S = [oracle.encode_planes(a, 1, q) for a in (vel, p0, p0)]
    pl = _plan(nx, ny, nz, n, k, codec="blockquant", rate=rate, stencil="star7")
    for a in range(3):
        pl.write_raw(a, S[a], 0, az)
    pl.run(k)
    got = pl.store(2, 0, az).astype(np.float64)
    got_raw = pl.read_raw(2, 0, az)
    pl.close()
    oracle.pipeline(ax, ay, nz, n, k, dt, k, 1, q, *S, stencil=oracle.STENCIL_STAR7)
    want = oracle.decode_planes(S[2], ax, ay, az, 1, q).astype(np.float64)
    rec = 8 * rate
    recs_g, recs_o = got_raw.reshape(-1, rec), S[2].reshape(-1, rec)
    same = np.all(recs_g == recs_o, axis=1).mean()
    # one quantisation step of the block (plus the stencil's tolerance) bounds every difference
    assert np.max(np.abs(got - want)) <= 2.0 ** -q * 2 * (np.abs(want).max() + 1e-30) + 1e-6
    assert same >= 0.5, same


def test_cfl_check_at_load():
    nx, ny, nz = 32, 16, 32
    vel, p0 = synth.fields(nx, ny, nz)
    vmax = float(np.abs(vel).max())
    az = vel.shape[0]
    limit = 2 / (3 * 2048 / 315) ** 0.5
    ok_dt, bad_dt = 0.99 * limit / vmax, 1.01 * limit / vmax
    for codec in ("identity", "blockquant"):
        pl = _plan(nx, ny, nz, 2, 1, codec=codec)  # dt from synth: CFL 0.4
        pl.load(0, vel, 0, az)
        pl.close()
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=bad_dt, n_blocks=2, tb_depth=1, codec=codec, mode="swb")
        pl = oocs.Plan(c)
        with pytest.raises(oocs.OocsError) as e:
            pl.load(0, vel, 0, az)
        assert e.value.status == 2 and "CFL" in str(e.value)
        pl.load(1, p0, 0, az)  # pressures are not velocity: no CFL check
        v2 = vel.copy()
        v2[5, 5, 5] = np.nan
        if codec == "identity":  # NaN velocity counts as above the limit (the lossy codec reports DATA first)
            with pytest.raises(oocs.OocsError):
                pl.load(0, v2, 0, az)
        pl.close()
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=ok_dt, n_blocks=2, tb_depth=1, codec=codec, mode="swb")
        pl = oocs.Plan(c)
        pl.load(0, vel, 0, az)
        # STAR7's limit is larger: bad_dt passes there
        pl.close()
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=bad_dt, n_blocks=2, tb_depth=1, codec=codec, mode="swb",
                             stencil="star7")
        pl = oocs.Plan(c)
        pl.load(0, vel, 0, az)
        pl.close()


def test_ext_streams_order_and_results():
    nx, ny, nz, n, k = 64, 32, 64, 4, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az = p0.shape[0]
    ref = _plan(nx, ny, nz, n, k, codec="blockquant")
    load_fields(ref, vel, p0)
    ref.run(2 * k)
    want = ref.read_raw(2, 0, az)
    ref.close()
    streams = [torch.cuda.Stream() for _ in range(3)]
    for executor in ("dispatch", "single", "split"):
        pl = _plan(nx, ny, nz, n, k, codec="blockquant", executor=executor,
                   ext_streams=[s.cuda_stream for s in streams])
        load_fields(pl, vel, p0)
        # work the caller queued on a lane's stream runs before the lane's kernels: a ~0.3 s sleep on
        # stream 0 delays the run's completion by at least that much
        with torch.cuda.stream(streams[0]):
            torch.cuda._sleep(int(0.3 * 1.9e9))
        t0 = time.perf_counter()
        pl.run(2 * k)
        dt_run = time.perf_counter() - t0
        assert dt_run >= 0.25, dt_run
        assert streams[0].query()  # the sleep is over by the time oocs_run returns
        assert np.array_equal(pl.read_raw(2, 0, az), want)
        pl.close()
    for s in streams:  # the plan did not destroy the caller's streams
        s.synchronize()


def test_cfl_check_at_load_device():
    nx, ny, nz = 32, 16, 32
    vel, p0 = synth.fields(nx, ny, nz)
    az = vel.shape[0]
    bad_dt = 1.01 * (2 / (3 * 2048 / 315) ** 0.5) / float(np.abs(vel).max())
    pl = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=bad_dt, n_blocks=2, tb_depth=1, mode="swb",
                                    store="device"))
    tv = torch.from_numpy(vel).cuda()
    with pytest.raises(oocs.OocsError) as e:
        pl.load_device(0, tv, 0, az)
    assert e.value.status == 2
    pl.load_device(1, torch.from_numpy(p0).cuda(), 0, az)
    pl.close()


@pytest.mark.parametrize("codec,rate", [("zfp", 12), ("trunc16", 16)])
def test_star7_other_codecs_pipeline_vs_oracle(codec, rate):
    """STAR7 through the ZFP / Truncate-16 pipelines: the GPU's S_T against the oracle pipeline's (same
    codec, same stencil) within the codec's own error after one sweep."""
    nx, ny, nz, n, k = 44, 20, 48, 3, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = p0.shape
    dt = synth.dt_for()
    cid, prm = {"zfp": (2, rate), "trunc16": (3, 0)}[codec]
    S = [oracle.encode_planes(a, cid, prm) for a in (vel, p0, p0)]
    pl = _plan(nx, ny, nz, n, k, codec=codec, rate=rate, stencil="star7")
    for a in range(3):
        pl.write_raw(a, S[a], 0, az)
    pl.run(k)
    got = pl.store(2, 0, az).astype(np.float64)
    pl.close()
    oracle.pipeline(ax, ay, nz, n, k, dt, k, cid, prm, *S, stencil=oracle.STENCIL_STAR7)
    want = oracle.decode_planes(S[2], ax, ay, az, cid, prm).astype(np.float64)
    amax = np.abs(want).max()
    tol = (2e-3 if codec == "zfp" else 2 ** -7) * amax
    assert np.max(np.abs(got - want)) <= tol
