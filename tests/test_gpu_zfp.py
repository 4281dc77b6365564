"""NEXT-1 on the GPU: the ZFP fixed-rate codec kernels against the oracle (bit-exact bitstream and
bitwise decode for identical input blocks), and the out-of-core pipeline with ZFP equal -- bitwise -- to
the same physics composed from the library's own kernels as in-core steps with a whole-field ZFP round
trip after every k steps (S:L467's injected-round-trip formulation, which the oracle pipeline also
satisfies: tests/test_oracle_zfp.py)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from test_gpu_parity import from_ws, stream, to_ws  # noqa: E402

R = 4
ZFP = 2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def gpu_encode(arr, rate):
    planes, ay, ax = arr.shape
    ws = to_ws(arr)
    out = torch.zeros(oracle.plane_bytes(ax, ay, ZFP, rate) * planes, dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    oocs.oocs_encode(ws.data_ptr(), out.data_ptr(), ax, ay, planes, oocs.pitch_for(ax), ZFP, rate, err.data_ptr(),
                     stream())
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    return out.cpu().numpy()


def gpu_decode(buf, ax, ay, planes, rate):
    src = torch.from_numpy(np.ascontiguousarray(buf)).cuda()
    ws = torch.full((planes, ay, oocs.pitch_for(ax)), float("nan"), dtype=torch.float32, device="cuda")
    oocs.oocs_decode(src.data_ptr(), ws.data_ptr(), ax, ay, planes, oocs.pitch_for(ax), ZFP, rate, stream())
    torch.cuda.synchronize()
    return from_ws(ws, ax)


@pytest.mark.parametrize("rate", [1, 2, 3, 4, 6, 8, 12, 16, 20, 24, 31, 32])
def test_zfp_bitstream_bit_exact(rate):
    planes, ay, ax = 8, 12, 44
    blocks = synth.random_blocks(planes * ay * ax // 64, seed=rate)
    arr = blocks.reshape(planes // 4, ay // 4, ax // 4, 4, 4, 4).transpose(0, 3, 1, 4, 2, 5).reshape(planes, ay, ax)
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    want = oracle.encode_planes(arr, ZFP, rate)
    got = gpu_encode(arr, rate)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:8]
    assert np.array_equal(gpu_decode(want, ax, ay, planes, rate).view(np.uint32),
                          oracle.decode_planes(want, ax, ay, planes, ZFP, rate).view(np.uint32))
    vel, p0 = synth.fields(64, 64, 32)
    for a in (vel[:16], p0[12:28]):
        a = np.ascontiguousarray(a)
        enc = oracle.encode_planes(a, ZFP, rate)
        assert np.array_equal(gpu_encode(a, rate), enc)
        # decode of smooth-field records (long zero runs, late significance) bitwise
        pl, ay2, ax2 = a.shape
        assert np.array_equal(gpu_decode(enc, ax2, ay2, pl, rate).view(np.uint32),
                              oracle.decode_planes(enc, ax2, ay2, pl, ZFP, rate).view(np.uint32))


@pytest.mark.parametrize("rate", [1, 2, 5, 16, 32])
def test_zfp_decode_arbitrary_records(rate):
    """The decoder's parser on arbitrary bit strings (every record is a valid fixed-rate stream): random
    words, words with sparse ones (long zero runs across word boundaries, runs cut by the budget or by
    position 63), all-ones -- bitwise equal to the oracle's decoder."""
    planes, ay, ax = 4, 8, 32
    nrec = (ay // 4) * (ax // 4) * (planes // 4)
    rng = np.random.default_rng(rate)
    words = rng.integers(0, 2**32, size=(nrec, 2 * rate), dtype=np.uint64).astype(np.uint32)
    sparse = rng.random((nrec, 2 * rate, 32)) < 0.02
    words[nrec // 3: 2 * nrec // 3] = (sparse[nrec // 3: 2 * nrec // 3] << np.arange(32)).sum(-1).astype(np.uint32)
    words[-2:] = 0xFFFFFFFF
    words[:, 0] |= 1  # non-zero blocks
    words[:, 0] = (words[:, 0] & ~np.uint32(0x1FE)) | (np.uint32(127 + 3) << 1)  # emax = 3: finite values
    buf = words.view(np.uint8).reshape(-1)
    got = gpu_decode(buf, ax, ay, planes, rate)
    want = oracle.decode_planes(buf, ax, ay, planes, ZFP, rate)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("store,sched", [("host", "alg1"), ("device", "alg1"), ("host", "dag")])
@pytest.mark.parametrize("rate,k", [(16, 2), (8, 1)])
def test_zfp_pipeline_equals_injected_roundtrip(store, sched, rate, k):
    nx, ny, nz, n = 40, 32, 64, 4
    vel, p0 = synth.fields(nx, ny, nz)
    az, ay, ax = vel.shape
    dt = synth.dt_for()
    T = 3 * k
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(dt), n_blocks=n, tb_depth=k, codec="zfp", rate_bits=rate,
                         mode="swb", store=store, schedule=sched)
    pl = oocs.Plan(c)
    for a, arr in enumerate((vel, p0, p0)):
        pl.load(a, arr, 0, az)
    pl.run(T)
    got = [pl.read_raw(a, 0, az) for a in (1, 2)]
    pl.close()
    # the same physics from the library's kernels: round trip, k whole-field steps, round trip, ...
    rt = lambda x: gpu_decode(gpu_encode(x, rate), ax, ay, az, rate)
    v, pp, pc = rt(vel), rt(p0), rt(p0)
    tv = to_ws(v)
    for _ in range(T // k):
        ta, tb = to_ws(pp), to_ws(pc)
        for _ in range(k):
            oocs.oocs_step(tv.data_ptr(), ta.data_ptr(), tb.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                           stream())
            ta, tb = tb, ta
        torch.cuda.synchronize()
        pp, pc = from_ws(ta, ax), from_ws(tb, ax)
        pp_b, pc_b = gpu_encode(pp, rate), gpu_encode(pc, rate)
        pp, pc = gpu_decode(pp_b, ax, ay, az, rate), gpu_decode(pc_b, ax, ay, az, rate)
    assert np.array_equal(got[0], pp_b) and np.array_equal(got[1], pc_b)


def test_zfp_gpu_matches_hand_derived_golden_records():
    """The GPU encoder against the records derived by hand in docs/FORMAT.md §4.1
    (tests/golden/zfp_blocks.txt), independently of the oracle: each golden block is placed at every
    position of a 4-plane slab of 3 x 3 blocks, encoded, and every record compared; decode is exact."""
    from test_oracle_zfp import golden_zfp_records

    for name, rate, x, want in golden_zfp_records():
        blk = x.reshape(4, 4, 4)  # (zi, yi, xi)
        arr = np.ascontiguousarray(np.tile(blk, (1, 3, 3)), dtype=np.float32)  # 4 planes x 12 x 12
        got = gpu_encode(arr, rate)
        rec = 8 * rate
        for i in range(9):
            assert got[i * rec:(i + 1) * rec].tobytes() == want, (name, rate, i)
        dec = gpu_decode(got, 12, 12, 4, rate)
        assert np.array_equal(dec.view(np.uint32), arr.view(np.uint32)), (name, rate)
