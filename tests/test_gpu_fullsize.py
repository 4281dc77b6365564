"""Parity at BASELINE.json's full size, in the launch configuration bench.py times.

configs[1] (c2): 1024^3 fp32, 8 chunks, k = 4, rate 16, single working buffer, state in HBM (bench `value`)
and in pinned host memory (bench `e2e`).  The CPU oracle cannot run 1.7e10 cell-updates in seconds, so it
recomputes sampled 4x4x4 output blocks one by one: for each sample it decodes the GPU's own input
bitstream S_0 around the block (the dependency cone, +-kR cells; the fixed Dirichlet halo where the cone
meets the domain edge), runs k in-core steps (temporal blocking validity makes the chunk's owned planes
equal to the in-core result), encodes the block and compares it with the GPU's record.  Byte counters are
checked against the fixed-rate transfer identities.  The same for the ZFP (NEXT-1) and
Truncate-16 codecs at rate 16."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4
NX, NY, NZ, NB, K, T, RATE = bench.WORKLOADS["c2"]
Q = RATE - 1


CODECS = {"blockquant": (1, Q), "zfp": (2, RATE), "trunc16": (3, 0)}  # oracle codec id, parameter


@pytest.fixture(scope="module", params=["blockquant", "zfp", "trunc16"])
def plans(request):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    dt = float(synth.dt_for())
    codec = request.param
    mk = lambda store: oocs.Plan(oocs.make_config(nx=NX, ny=NY, nz=NZ, dt=dt, n_blocks=NB, tb_depth=K,
                                                  rate_bits=RATE, mode="swb", store=store, codec=codec,
                                                  n_lanes=2))  # bench.py --lanes 2
    dev = mk("device")
    bench.load_state(dev, NX, NY, NZ, 0)
    host = mk("host")
    bench.copy_state(dev, host)
    az = NZ + 2 * R
    s0 = {a: dev.read_raw(a, 0, az) for a in range(3)}
    yield dev, host, s0, codec
    dev.close()
    host.close()


def _samples(rng, n):
    ax, ay, az = NX + 2 * R, NY + 2 * R, NZ + 2 * R
    nbx, nby, nbz = ax // 4, ay // 4, az // 4
    W = NZ // NB
    picks = [(1, 1, 1), (nbx - 2, nby - 2, nbz - 2), (nbx // 2, 1, (W + R) // 4), (1, nby // 2, (W + R) // 4 - 1),
             (nbx - 2, 3, (2 * W + R) // 4), (5, nby - 2, (3 * W + R) // 4 + 1)]  # edges and chunk seams
    while len(picks) < n:
        picks.append((int(rng.integers(1, nbx - 1)), int(rng.integers(1, nby - 1)), int(rng.integers(1, nbz - 1))))
    return picks


def _oracle_block(s0, bx, by, bz, dt, codec="blockquant"):
    """Oracle value of interior block (bx, by, bz) (allocated block coords) after K steps: levels K-1, K."""
    ax, ay, az = NX + 2 * R, NY + 2 * R, NZ + 2 * R
    m = K * R
    lo = [max(0, 4 * b - m) for b in (bx, by, bz)]
    hi = [min(n, 4 * b + 4 + m) for b, n in ((bx, ax), (by, ay), (bz, az))]
    zl, zh = lo[2] // 4 * 4, (hi[2] + 3) // 4 * 4
    cid, prm = CODECS[codec]
    pb = oracle.plane_bytes(ax, ay, cid, prm)
    sub = []
    for a in range(3):
        full = oracle.decode_planes(s0[a][zl * pb:zh * pb], ax, ay, zh - zl, cid, prm)
        sub.append(np.ascontiguousarray(full[lo[2] - zl:hi[2] - zl, lo[1]:hi[1], lo[0]:hi[0]]))
    v, pp, pc = sub
    pp, pc = oracle.incore(v, pp, pc, dt, K)
    sl = (slice(4 * bz - lo[2], 4 * bz - lo[2] + 4), slice(4 * by - lo[1], 4 * by - lo[1] + 4),
          slice(4 * bx - lo[0], 4 * bx - lo[0] + 4))
    return pp[sl], pc[sl]


@pytest.mark.parametrize("store", ["device", "host"])
def test_c2_sampled_blocks_after_one_sweep(plans, store):
    dev, host, s0, codec = plans
    pl = dev if store == "device" else host
    az, ax, ay = NZ + 2 * R, NX + 2 * R, NY + 2 * R
    for a in range(3):  # every store starts from the same S_0
        pl.write_raw(a, s0[a], 0, az)
    st = pl.run(K)
    # fixed-rate transfer identities (host store): H2D = 3 arrays x (nz + 2R) planes, D2H = 2 x nz planes
    pb = pl.info.plane_bytes
    if store == "host":
        assert st.bytes_h2d == 3 * (NZ + 2 * R) * pb
        assert st.bytes_d2h == 2 * NZ * pb
    assert st.cell_updates == NX * NY * NZ * K
    dt = synth.dt_for()
    rng = np.random.default_rng(2204)
    samples = _samples(rng, 16)
    if codec != "blockquant":
        _check_other_codec(pl, s0, codec, samples, dt)
        return
    nbx, nby = ax // 4, ay // 4
    rec = 8 * (Q + 1)
    exact = 0
    for (bx, by, bz) in samples:
        want_p, want_c = _oracle_block(s0, bx, by, bz, dt)
        for arr, want in ((1, want_p), (2, want_c)):
            slab = pl.read_raw(arr, 4 * bz, 4 * bz + 4)
            r = slab[(by * nbx + bx) * rec:(by * nbx + bx + 1) * rec].tobytes()
            got = oracle.decode_block(r, Q).reshape(4, 4, 4)
            ref_rec = oracle.encode_block(np.ascontiguousarray(want).reshape(64), Q)
            exact += r == ref_rec
            ref = oracle.decode_block(ref_rec, Q).reshape(4, 4, 4).astype(np.float64)
            mn, mx = np.frombuffer(ref_rec[:8], dtype=np.float32)
            step = (float(mx) - float(mn)) / 2 ** Q
            tol = 1.01 * step + K * 1e-6 * max(np.abs(ref).max(), 1e-30) + 4 * np.spacing(np.float32(np.abs(ref).max()))
            assert np.all(np.abs(got - ref) <= tol), (bx, by, bz, arr)
    assert exact >= len(samples)  # most records are bit-identical (codes flip only at bin edges)


def _check_other_codec(pl, s0, codec, samples, dt):
    """ZFP / Truncate-16: decode the GPU's 4-plane slab around each sampled block and compare the block
    with the oracle's k in-core steps from the same S_0, within the codec's own error on the oracle's
    values (ZFP: twice its measured round-trip error; bf16: one ulp) plus the stencil's 1e-6 per step."""
    ax, ay = NX + 2 * R, NY + 2 * R
    cid, prm = CODECS[codec]
    exact = n = 0
    for (bx, by, bz) in samples:
        want_p, want_c = _oracle_block(s0, bx, by, bz, dt, codec)
        for arr, want in ((1, want_p), (2, want_c)):
            slab = pl.read_raw(arr, 4 * bz, 4 * bz + 4)
            got = oracle.decode_planes(slab, ax, ay, 4, cid, prm)[:, 4 * by:4 * by + 4, 4 * bx:4 * bx + 4]
            want = np.ascontiguousarray(want, dtype=np.float32)
            amax = max(float(np.abs(want).max()), 1e-30)
            stencil = K * 1e-6 * amax
            if codec == "zfp":
                # the oracle's record of its own result for this block, via a 4-plane slab holding it
                tile = np.zeros((4, 4, 4), dtype=np.float32)
                tile[:] = want
                ref_rec = oracle.zfp_encode_block(tile.reshape(64), RATE)
                ref = oracle.zfp_decode_block(ref_rec, RATE).reshape(4, 4, 4)
                rec_bytes = 8 * RATE
                nbx = ax // 4
                exact += slab[(by * nbx + bx) * rec_bytes:(by * nbx + bx + 1) * rec_bytes].tobytes() == ref_rec
                err = float(np.abs(ref.astype(np.float64) - want).max())
                tol = 2 * err + 4 * stencil + 4 * np.spacing(np.float32(amax))
            else:
                ref = oracle.decode_planes(oracle.encode_planes(want, cid, prm), 4, 4, 4, cid, prm)
                exact += np.array_equal(ref.view(np.uint32), got.view(np.uint32))
                ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(want.astype(np.float64)), 1e-38))) - 7)
                tol = ulp + stencil
            n += 1
            assert np.all(np.abs(got.astype(np.float64) - want) <= tol), (codec, bx, by, bz, arr)
    # Truncate-16 records are bit-identical unless a bf16 rounding boundary was straddled.  ZFP records
    # mostly differ in low bit planes: the stencil's (normwise 1e-6) fp32 differences are relative to
    # the block's own scale in small-valued blocks, and every coded plane of a block carries them
    if codec == "trunc16":
        assert exact >= n // 2, (codec, exact, n)
