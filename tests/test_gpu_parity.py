"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north star in BASELINE.json): compressed bitstream bit-exact for
identical input blocks; stencil within max relative error 1e-6 per step
(Q16: max|g-o| / max|o| over the updated region); out-of-core runs
compared with the oracle pipeline (bitwise with the identity codec, within one
quantisation step per sweep with the lossy codec -- DESIGN.md §5).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4
XOFF = oocs.XOFF


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def to_ws(arr: np.ndarray) -> "torch.Tensor":
    """(planes, ay, ax) float32 -> device working-buffer layout (planes, ay, pitch), data at col XOFF."""
    planes, ay, ax = arr.shape
    pitch = oocs.pitch_for(ax)
    buf = np.zeros((planes, ay, pitch), dtype=np.float32)
    buf[:, :, XOFF:XOFF + ax] = arr
    return torch.from_numpy(buf).cuda()


def from_ws(t: "torch.Tensor", ax: int) -> np.ndarray:
    return np.ascontiguousarray(t.cpu().numpy()[:, :, XOFF:XOFF + ax])


def stream():
    return torch.cuda.current_stream().cuda_stream


def gpu_encode(arr: np.ndarray, codec: int, rate: int) -> np.ndarray:
    planes, ay, ax = arr.shape
    ws = to_ws(arr)
    q = rate - 1
    nbytes = oracle.plane_bytes(ax, ay, codec, q) * planes
    out = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    oocs.oocs_encode(ws.data_ptr(), out.data_ptr(), ax, ay, planes, oocs.pitch_for(ax), codec, rate,
                     err.data_ptr(), stream())
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    return out.cpu().numpy()


def gpu_decode(buf: np.ndarray, ax, ay, planes, codec, rate) -> np.ndarray:
    src = torch.from_numpy(np.ascontiguousarray(buf)).cuda()
    ws = torch.full((planes, ay, oocs.pitch_for(ax)), float("nan"), dtype=torch.float32, device="cuda")
    oocs.oocs_decode(src.data_ptr(), ws.data_ptr(), ax, ay, planes, oocs.pitch_for(ax), codec, rate, stream())
    torch.cuda.synchronize()
    return from_ws(ws, ax)


# ----------------------------------------------------------------------------- codec
@pytest.mark.parametrize("rate", [2, 8, 12, 16, 17, 24])
@pytest.mark.parametrize("shape", [(8, 12, 44), (4, 40, 72), (12, 8, 164)])
def test_codec_bitstream_bit_exact(rate, shape):
    rng = np.random.default_rng(rate * 1000 + shape[2])
    planes, ay, ax = shape
    blocks = synth.random_blocks(planes * ay * ax // 64, seed=rate + shape[2])
    arr = blocks.reshape(planes // 4, ay // 4, ax // 4, 4, 4, 4).transpose(0, 3, 1, 4, 2, 5).reshape(shape)
    arr = np.ascontiguousarray(arr * rng.choice([1.0, -1.0], size=1)[0], dtype=np.float32)
    want = oracle.encode_planes(arr, oracle.CODEC_BLOCKQUANT, rate - 1)
    got = gpu_encode(arr, 1, rate)
    assert got.shape == want.shape
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    # decode: identical bytes in -> identical floats out (bitwise)
    d_gpu = gpu_decode(want, ax, ay, planes, 1, rate)
    d_ora = oracle.decode_planes(want, ax, ay, planes, 1, rate - 1)
    assert np.array_equal(d_gpu.view(np.uint32), d_ora.view(np.uint32))


def test_codec_on_paper_like_fields_and_identity():
    vel, p0 = synth.fields(64, 64, 64)
    for arr in (vel[:32], p0[20:52]):
        arr = np.ascontiguousarray(arr)
        for rate in (8, 16, 24):
            assert np.array_equal(gpu_encode(arr, 1, rate), oracle.encode_planes(arr, 1, rate - 1))
        raw = gpu_encode(arr, 0, 32)
        assert raw.tobytes() == arr.tobytes()
        assert np.array_equal(gpu_decode(raw, 72, 72, 32, 0, 32), arr)


@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan, -np.nan, 2.0 ** 126, -(2.0 ** 127)])
@pytest.mark.parametrize("rate", [8, 16, 24])
def test_encoder_flags_nonfinite(bad, rate):
    """a lossy encode of NaN, +-Inf or |x| >= 2^126 raises the error flag -- wherever in the
    4x4x4 block (every value position, i.e. every lane/row of the warp layout) and in any block of the
    line; an all-finite input does not."""
    ax, ay, planes = 40, 8, 4
    rng = np.random.default_rng(rate)
    for pos in range(0, 64 * (ax // 4), 7):
        arr = rng.standard_normal((planes, ay, ax)).astype(np.float32)
        b, j = divmod(pos, 64)
        zi, yi, xi = j // 16, (j // 4) % 4, j % 4
        arr[zi, yi, 4 * b + xi] = bad
        ws = to_ws(arr)
        out = torch.zeros(oracle.plane_bytes(ax, ay, 1, rate - 1) * planes, dtype=torch.uint8, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        oocs.oocs_encode(ws.data_ptr(), out.data_ptr(), ax, ay, planes, oocs.pitch_for(ax), 1, rate,
                         err.data_ptr(), stream())
        torch.cuda.synchronize()
        assert int(err.item()) == 1, (bad, pos)
    arr = rng.standard_normal((planes, ay, ax)).astype(np.float32)
    gpu_encode(arr, 1, rate)  # asserts the flag stays 0


# ----------------------------------------------------------------------------- stencil
def _rel_err(g, o):
    return np.max(np.abs(g.astype(np.float64) - o)) / np.max(np.abs(o))


@pytest.mark.parametrize("nx,ny,nz", [(64, 64, 24), (44, 36, 16), (12, 100, 12), (96, 8, 40)])
def test_stencil_step_within_1e6(nx, ny, nz):
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(nx + ny)
    pprev = (p0 * np.float32(0.97) + rng.normal(scale=1e-3, size=p0.shape).astype(np.float32))
    pprev[:R], pprev[-R:], pprev[:, :R], pprev[:, -R:], pprev[:, :, :R], pprev[:, :, -R:] = 0, 0, 0, 0, 0, 0
    pprev = np.ascontiguousarray(pprev, dtype=np.float32)
    dt = synth.dt_for()
    az, ay, ax = p0.shape
    for (zlo, zhi) in [(R, az - R), (R + 3, az - R - 5)]:
        o = pprev.copy()
        oracle.step(vel, o, p0, dt, zlo, zhi)
        tv, tp, tc = to_ws(vel), to_ws(pprev), to_ws(p0)
        oocs.oocs_step(tv.data_ptr(), tp.data_ptr(), tc.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, zlo, zhi,
                       stream())
        torch.cuda.synchronize()
        g = from_ws(tp, ax)
        sl = (slice(zlo, zhi), slice(R, ay - R), slice(R, ax - R))
        assert _rel_err(g[sl], o[sl].astype(np.float64)) <= 1e-6
        # untouched outside the region (incl. the Dirichlet halo), bitwise
        mask = np.ones(g.shape, dtype=bool)
        mask[sl] = False
        assert np.array_equal(g[mask].view(np.uint32), pprev[mask].view(np.uint32))
        # GPU in-padding columns are never written either
        full = tp.cpu().numpy()
        assert np.all(full[:, :, :XOFF] == 0) and np.all(full[:, :, XOFF + ax:] == 0)


def _ulp_distance(g: np.ndarray, o: np.ndarray) -> np.ndarray:
    """Per-element distance in fp32 ulps (ordered-integer difference of the bit patterns)."""
    def ordered(a):
        i = a.astype(np.float32).view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    return np.abs(ordered(g) - ordered(o))


def test_stencil_ulp_histogram():
    """SURVEY Q16 beside the normwise 1e-6 bar: the per-element distance, in fp32 ulps, between the GPU
    step (fp32, difference form, FMA chain) and the oracle step (fp64, one rounding) on the synthetic
    fields over a grid spanning several CTA tiles (64 x 16) and a ragged tail.  Written to
    $OOCS_REPORT_DIR/stencil_ulp_hist.json for profiles/."""
    import json
    import os
    nx, ny, nz = 200, 72, 40
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(7)
    pprev = (p0 * np.float32(0.97) + rng.normal(scale=1e-3, size=p0.shape).astype(np.float32))
    pprev[:R], pprev[-R:], pprev[:, :R], pprev[:, -R:], pprev[:, :, :R], pprev[:, :, -R:] = 0, 0, 0, 0, 0, 0
    pprev = np.ascontiguousarray(pprev, dtype=np.float32)
    dt = synth.dt_for()
    az, ay, ax = p0.shape
    o = pprev.copy()
    oracle.step(vel, o, p0, dt, R, az - R)
    tv, tp, tc = to_ws(vel), to_ws(pprev), to_ws(p0)
    oocs.oocs_step(tv.data_ptr(), tp.data_ptr(), tc.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                   stream())
    torch.cuda.synchronize()
    g = from_ws(tp, ax)
    sl = (slice(R, az - R), slice(R, ay - R), slice(R, ax - R))
    d = _ulp_distance(g[sl], o[sl]).ravel()
    edges = [0, 1, 2, 3, 5, 9, 17, 65, 1 << 62]
    counts = np.histogram(d, bins=edges)[0].tolist()
    rel = _rel_err(g[sl], o[sl].astype(np.float64))
    hist = {"cells": int(d.size), "bins_ulp": ["0", "1", "2", "3-4", "5-8", "9-16", "17-64", ">64"],
            "counts": counts, "median_ulp": float(np.median(d)), "p99_ulp": float(np.percentile(d, 99)),
            "max_ulp": int(d.max()), "normwise_rel_err": rel,
            "note": "large ulp counts occur only where p_next is small against its terms (cancellation); "
                    "the bar is the normwise 1e-6"}
    out = os.environ.get("OOCS_REPORT_DIR", os.path.join(os.path.dirname(os.path.dirname(__file__)), "gpurun_out"))
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "stencil_ulp_hist.json"), "w") as f:
        json.dump(hist, f, indent=1)
    assert rel <= 1e-6
    assert hist["median_ulp"] <= 1.0


# ----------------------------------------------------------------------------- out-of-core runs
def make_plan(nx, ny, nz, n, k, codec="blockquant", rate=16, mode="swb", store="host", profile=False,
              resident_velocity=False, n_lanes=0, schedule="alg1", executor="dispatch"):
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, codec=codec,
                         rate_bits=rate, mode=mode, store=store, profile=profile,
                         resident_velocity=resident_velocity, n_lanes=n_lanes, schedule=schedule,
                         executor=executor)
    return oocs.Plan(c)


def load_fields(plan, vel, p0):
    az = vel.shape[0]
    plan.load(0, vel, 0, az)
    plan.load(1, p0, 0, az)
    plan.load(2, p0, 0, az)


IDENTITY_MODES = [("baseline", "host", "alg1"), ("compress", "host", "alg1"), ("swb", "host", "alg1"),
                  ("dwb", "host", "alg1"), ("swb", "device", "alg1"), ("baseline", "host", "dag_func"),
                  ("swb", "host", "dag")]


@pytest.mark.parametrize("n,k", [(4, 2), (3, 1), (2, 3), (1, 2)])
def test_identity_pipeline_bitwise_all_modes_and_vs_oracle(n, k):
    nx, ny, nz = 44, 36, 96
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    T = 2 * k
    results = []
    for mode, store, sched in IDENTITY_MODES:
        pl = make_plan(nx, ny, nz, n, k, codec="identity", mode=mode, store=store, schedule=sched)
        load_fields(pl, vel, p0)
        st = pl.run(T)
        results.append((pl.store(1, 0, az), pl.store(2, 0, az)))
        assert st.cell_updates == nx * ny * nz * T
        pl.close()
    for pp, pc in results[1:]:
        assert np.array_equal(pp.view(np.uint32), results[0][0].view(np.uint32))
        assert np.array_equal(pc.view(np.uint32), results[0][1].view(np.uint32))
    # vs the oracle in-core run (fp64 arithmetic): per-step tolerance accumulated over T steps
    _, oc = oracle.incore(vel, p0.copy(), p0.copy(), synth.dt_for(), T)
    assert _rel_err(results[0][1], oc.astype(np.float64)) <= 1e-6 * T


def test_identity_pipeline_equals_gpu_incore():
    nx, ny, nz = 32, 32, 64
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    T = 4
    pl = make_plan(nx, ny, nz, 4, 2, codec="identity", mode="swb")
    load_fields(pl, vel, p0)
    pl.run(T)
    got = pl.store(2, 0, az)
    tv, ta, tb = to_ws(vel), to_ws(p0), to_ws(p0)
    for _ in range(T):
        oocs.oocs_step(tv.data_ptr(), ta.data_ptr(), tb.data_ptr(), ax, ay, az, oocs.pitch_for(ax),
                       synth.dt_for(), R, az - R, stream())
        ta, tb = tb, ta
    torch.cuda.synchronize()
    assert np.array_equal(from_ws(tb, ax).view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("rate", [8, 16, 24])
def test_lossy_modes_are_bitwise_identical(rate):
    nx, ny, nz = 40, 32, 64
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    outs = []
    variants = [("compress", "host", False, 0, "alg1"), ("swb", "host", False, 0, "alg1"),
                ("dwb", "host", False, 0, "alg1"), ("swb", "device", False, 0, "alg1"),
                ("swb", "host", True, 0, "alg1"), ("swb", "host", False, 4, "alg1"), ("dwb", "host", True, 2, "alg1"),
                ("swb", "host", False, 0, "dag"), ("swb", "host", False, 0, "dag_func"),
                ("compress", "host", True, 4, "dag_func")]
    # the same schedules replayed onto streams (one per lane, Alg. 1 literally / copy + kernel per lane)
    # instead of the host dispatcher
    variants += [v + (ex,) for ex in ("single", "split") for v in variants[:4] + variants[6:8]]
    variants += [("swb", "host", False, 2, "alg1")]  # the bench's out-of-core configuration (2 lanes)
    # the by-function DAG schedule runs three streams whatever the lane count (n_lanes = 2 once crashed)
    variants += [("swb", "host", False, 2, "dag_func"), ("swb", "host", True, 2, "dag_func", "single"),
                 ("dwb", "host", False, 2, "dag_func", "split")]
    for mode, store, resident, lanes, sched, *ex in variants:
        pl = make_plan(nx, ny, nz, 4, 2, rate=rate, mode=mode, store=store, resident_velocity=resident,
                       n_lanes=lanes, schedule=sched, executor=ex[0] if ex else "dispatch")
        load_fields(pl, vel, p0)
        pl.run(6)
        outs.append((pl.read_raw(1, 0, az), pl.read_raw(2, 0, az)))
        pl.close()
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


def _block_steps(rec_bytes, q, nblk):
    recs = rec_bytes.reshape(nblk, 8 * (q + 1))
    mn = recs[:, 0:4].copy().view(np.float32)[:, 0].astype(np.float64)
    mx = recs[:, 4:8].copy().view(np.float32)[:, 0].astype(np.float64)
    return (mx - mn) / 2.0 ** q


@pytest.mark.parametrize("n,k,rate", [(4, 2, 16), (3, 1, 8), (2, 3, 24)])
def test_lossy_sweep_parity_vs_oracle(n, k, rate):
    """Per sweep: identical compressed S_t on both sides -> one sweep -> decoded S_{t+1} agree within
    one quantisation step of the block (+4 ulp): codes may differ by one only where the stencil's
    fp32 rounding (<= 1e-6 relative) straddles a bin edge; the bitstreams must otherwise agree."""
    q = rate - 1
    nx, ny, nz = 44, 40, 96
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    S = [oracle.encode_planes(a, 1, q) for a in (vel, p0, p0)]
    pl = make_plan(nx, ny, nz, n, k, rate=rate)
    dt = synth.dt_for()
    for a in range(3):
        pl.write_raw(a, S[a], 0, az)
    for sweep in range(2):
        pl.run(k)
        Sp, Sc = S[1].copy(), S[2].copy()
        oracle.pipeline(ax, ay, nz, n, k, dt, k, 1, q, S[0], Sp, Sc)
        for a, Sref in ((1, Sp), (2, Sc)):
            g = pl.read_raw(a, 0, az)
            # fraction of differing bytes ~ (fp32 rounding gap) / step ~ 2^q * 1e-7: only meaningful at q <= 15
            if q <= 15:
                assert np.mean(g != Sref) < 0.02
            dg = oracle.decode_planes(g, ax, ay, az, 1, q).astype(np.float64)
            do = oracle.decode_planes(Sref, ax, ay, az, 1, q).astype(np.float64)
            nblk = g.size // (8 * (q + 1))
            step = _block_steps(Sref, q, nblk)
            # per-cell tolerance: the block's step, broadcast to its 64 cells
            tol = step.reshape(az // 4, ay // 4, ax // 4)
            tol = np.repeat(np.repeat(np.repeat(tol, 4, 0), 4, 1), 4, 2)
            amax = np.maximum(np.abs(dg), np.abs(do))
            # + the stencil's own per-step tolerance (1e-6 of max|o|, north star) over the k steps: at
            # q = 23 a quantisation step is below fp32 stencil rounding
            stencil_tol = k * 1e-6 * np.max(np.abs(do))
            assert np.all(np.abs(dg - do) <= tol * 1.01 + 4 * np.spacing(amax.astype(np.float32)) + stencil_tol)
        # continue both sides from the oracle's state (identical inputs each sweep)
        S[1], S[2] = Sp, Sc
        pl.write_raw(1, Sp, 0, az)
        pl.write_raw(2, Sc, 0, az)


def test_c1_end_to_end_error_report():
    """BASELINE configs[0]: 64^3, 4 blocks, 4 steps, k=2, rate 16: GPU vs oracle pipeline, and vs in-core."""
    nx = ny = nz = 64
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    q = 15
    pl = make_plan(nx, ny, nz, 4, 2, rate=16)
    load_fields(pl, vel, p0)
    pl.run(4)
    g = pl.store(2, 0, az).astype(np.float64)
    S = [oracle.encode_planes(a, 1, q) for a in (vel, p0, p0)]
    oracle.pipeline(ax, ay, nz, 4, 2, synth.dt_for(), 4, 1, q, *S)
    o = oracle.decode_planes(S[2], ax, ay, az, 1, q).astype(np.float64)
    _, ic = oracle.incore(vel, p0.copy(), p0.copy(), synth.dt_for(), 4)
    ic = ic.astype(np.float64)
    inner = (slice(R, -R),) * 3
    err_go = np.max(np.abs(g - o))
    err_gi = np.max(np.abs(g - ic))
    rmse = np.sqrt(np.mean((g[inner] - ic[inner]) ** 2))
    psnr = 20 * np.log10((ic[inner].max() - ic[inner].min()) / rmse)
    assert err_go < 1e-4
    assert err_gi < 1e-3 and psnr > 80


def test_device_oom_and_bad_steps():
    c = oocs.make_config(nx=64, ny=64, nz=64, dt=0.1, n_blocks=4, tb_depth=2, device_capacity=1 << 20)
    with pytest.raises(oocs.OocsError) as e:
        oocs.Plan(c)
    assert e.value.status == 3
    pl = make_plan(32, 32, 32, 2, 2)
    with pytest.raises(oocs.OocsError) as e:
        pl.run(3)
    assert e.value.status == 2
    bad = np.ones((40, 40, 40), dtype=np.float32)
    bad[7, 7, 7] = np.nan
    with pytest.raises(oocs.OocsError) as e:
        pl.load(1, bad, 0, 40)
    assert e.value.status == 6


def test_degenerate_cases():
    """steps = 0 leaves the state bitwise unchanged; the smallest legal grid (4^3 interior, 2 chunks of
    8 planes, k = 1); a single chunk spanning the whole domain; all with the lossy codec."""
    vel, p0 = synth.fields(4, 4, 16)
    az = 16 + 2 * R
    pl = make_plan(4, 4, 16, 2, 1, rate=16)
    load_fields(pl, vel, p0)
    before = pl.read_raw(2, 0, az)
    st = pl.run(0)
    assert st.cell_updates == 0 and np.array_equal(pl.read_raw(2, 0, az), before)
    pl.run(3)
    S = [oracle.encode_planes(a, 1, 15) for a in (vel, p0, p0)]
    oracle.pipeline(12, 12, 16, 2, 1, synth.dt_for(), 3, 1, 15, *S)
    got = oracle.decode_planes(pl.read_raw(2, 0, az), 12, 12, az, 1, 15)
    want = oracle.decode_planes(S[2], 12, 12, az, 1, 15)
    assert np.max(np.abs(got - want)) < 1e-4
    pl.close()
    # one chunk = the whole domain (no carry, both physical boundaries in one extent)
    vel, p0 = synth.fields(16, 16, 32)
    a1 = make_plan(16, 16, 32, 1, 2, codec="identity")
    load_fields(a1, vel, p0)
    a1.run(4)
    _, pc = oracle.incore(vel, p0.copy(), p0.copy(), synth.dt_for(), 4)
    assert _rel_err(a1.store(2, 0, 40), pc.astype(np.float64)) <= 4e-6
    a1.close()


@pytest.mark.parametrize("codec,rate", [("blockquant", 16), ("blockquant", 8), ("zfp", 12), ("trunc16", 16),
                                        ("identity", 32)])
def test_decoded_velocity_is_bitwise_identical(codec, rate):
    """OOCS_FLAG_DECODED_VELOCITY (device store): the stencil reads the velocity from a resident array
    decoded once at load instead of from each chunk's decode -- the same decode of the same records, so
    S_T is bitwise the same; reloading the velocity (load and write_raw) re-decodes it."""
    nx, ny, nz, n, k = 44, 36, 96, 4, 3
    vel, p0 = synth.fields(nx, ny, nz)
    vel2 = np.ascontiguousarray(vel[:, :, ::-1] * np.float32(0.9))
    az = nz + 2 * R
    outs = []
    for dec in (False, True):
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, codec=codec,
                             rate_bits=rate, mode="swb", store="device", decoded_velocity=dec)
        pl = oocs.Plan(c)
        load_fields(pl, vel, p0)
        pl.run(2 * k)
        o = [pl.read_raw(a, 0, az) for a in (1, 2)]
        pl.load(0, vel2, 0, az)  # a new velocity model mid-run
        pl.run(k)
        o += [pl.read_raw(a, 0, az) for a in (1, 2)]
        raw_v = pl.read_raw(0, 0, az)
        pl.write_raw(0, raw_v, 0, az)  # same bytes through write_raw: same result again
        pl.run(k)
        o += [pl.read_raw(a, 0, az) for a in (1, 2)]
        outs.append(o)
        pl.close()
    for i, (a, b) in enumerate(zip(*outs)):
        assert np.array_equal(a, b), (i, np.flatnonzero(a != b)[:8])
