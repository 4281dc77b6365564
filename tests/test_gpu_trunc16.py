"""Truncate-16 codec (OOCS_CODEC_TRUNC16) on the GPU against the oracle: the
bf16 bytes bit-exact for identical inputs (every exponent, rounding ties, subnormals, +-0, Inf, NaN,
random bit patterns and paper-like fields, ragged shapes), decode bitwise, the out-of-core pipeline
bitwise equal to in-core steps with an injected whole-field round trip after every sweep, and
one sweep from identical compressed state within half a bf16 ulp (+ the stencil's 1e-6) of the
oracle's pipeline."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from test_gpu_parity import from_ws, gpu_decode, gpu_encode, stream, to_ws  # noqa: E402

R = 4
C = 3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _special_bits(n):
    rng = np.random.default_rng(7)
    e = np.arange(256, dtype=np.uint32) << 23
    fr = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0x17FFF, 0x18000, 0x18001, 0x7FFFFF, 0x7F8000, 0x400001], np.uint32)
    grid = (e[:, None] | fr[None, :]).ravel()
    bits = np.concatenate([grid, grid | 0x80000000, rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)])
    return bits


@pytest.mark.parametrize("shape", [(4, 12, 12), (8, 36, 44), (12, 8, 164), (4, 100, 72)])
def test_trunc16_bit_exact(shape):
    planes, ay, ax = shape
    m = planes * ay * ax
    bits = np.resize(_special_bits(m), m)
    arr = bits.view(np.float32).reshape(shape)
    want = oracle.encode_planes(arr, C, 0)
    got = gpu_encode(arr, C, 16)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:8]
    assert np.array_equal(gpu_decode(want, ax, ay, planes, C, 16).view(np.uint32),
                          oracle.decode_planes(want, ax, ay, planes, C, 0).view(np.uint32))
    vel, p0 = synth.fields(max(ax - 2 * R, 4), max(ay - 2 * R, 4), 4 * planes)
    for a in (vel[:planes, :ay, :ax], p0[planes:2 * planes, :ay, :ax]):
        a = np.ascontiguousarray(a)
        assert np.array_equal(gpu_encode(a, C, 16), oracle.encode_planes(a, C, 0))


@pytest.mark.parametrize("store,sched,k", [("host", "alg1", 2), ("device", "alg1", 2), ("host", "dag", 1),
                                           ("device", "dag_func", 3)])
def test_trunc16_pipeline_equals_injected_roundtrip(store, sched, k):
    nx, ny, nz, n = 40, 32, 64, 4
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    dt = synth.dt_for()
    T = 3 * k
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(dt), n_blocks=n, tb_depth=k, codec="trunc16", rate_bits=16,
                         mode="swb", store=store, schedule=sched)
    pl = oocs.Plan(c)
    for a, arr in enumerate((vel, p0, p0)):
        pl.load(a, arr, 0, az)
    pl.run(T)
    got = [pl.read_raw(a, 0, az) for a in (1, 2)]
    pl.close()
    rt = lambda x: gpu_decode(gpu_encode(x, C, 16), ax, ay, az, C, 16)
    v, pp, pc = rt(vel), rt(p0), rt(p0)
    tv = to_ws(v)
    for _ in range(T // k):
        ta, tb = to_ws(pp), to_ws(pc)
        for _ in range(k):
            oocs.oocs_step(tv.data_ptr(), ta.data_ptr(), tb.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                           stream())
            ta, tb = tb, ta
        torch.cuda.synchronize()
        pp_b, pc_b = gpu_encode(from_ws(ta, ax), C, 16), gpu_encode(from_ws(tb, ax), C, 16)
        pp, pc = gpu_decode(pp_b, ax, ay, az, C, 16), gpu_decode(pc_b, ax, ay, az, C, 16)
    assert np.array_equal(got[0], pp_b) and np.array_equal(got[1], pc_b)


@pytest.mark.parametrize("n,k", [(4, 2), (3, 1)])
def test_trunc16_sweep_parity_vs_oracle(n, k):
    nx, ny, nz = 44, 40, 96
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    S = [oracle.encode_planes(a, C, 0) for a in (vel, p0, p0)]
    dt = synth.dt_for()
    pl = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(dt), n_blocks=n, tb_depth=k, codec="trunc16",
                                    rate_bits=16, mode="swb", store="host"))
    for a in range(3):
        pl.write_raw(a, S[a], 0, az)
    pl.run(k)
    Sp, Sc = S[1].copy(), S[2].copy()
    oracle.pipeline(ax, ay, nz, n, k, dt, k, C, 0, S[0], Sp, Sc)
    for a, Sref in ((1, Sp), (2, Sc)):
        g = pl.read_raw(a, 0, az)
        assert np.mean(g.view(np.uint16) != Sref.view(np.uint16)) < 0.01  # only rounding-boundary flips
        dg = oracle.decode_planes(g, ax, ay, az, C, 0).astype(np.float64)
        do = oracle.decode_planes(Sref, ax, ay, az, C, 0).astype(np.float64)
        ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(do), 1e-38))) - 7)  # one bf16 ulp
        assert np.all(np.abs(dg - do) <= ulp + k * 1e-6 * np.max(np.abs(do)))
    pl.close()
