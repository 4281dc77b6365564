"""Pins for the oracle's decomposition and out-of-core pipeline.

Plan: SPEC worked examples and brute-force coverage
(S:L94-95).  Pipeline: the temporal-blocking validity invariant (S:L160,
S:L500, acceptance #1 S:L654) -- with the identity codec the blocked
out-of-core result is bitwise the plain in-core result -- and, for the lossy
codec, bitwise equality with an independent formulation: in-core steps with a
whole-field compress/decompress round trip injected after every k steps
("oracle with an injected per-sweep truncation").
"""
import numpy as np
import pytest

import oracle
import synth

R = oracle.R


def test_plan_spec_example_table1():
    p = oracle.plan(1152, 8, 12)
    assert all(p[i, 1] - p[i, 0] == 144 for i in range(8))
    assert p[1, 2] == 144 - 48 and p[1, 3] == 288 + 48
    assert p[0, 3] - p[1, 2] == 96  # interior overlap width 2kR
    assert p[0, 2] == -R and p[7, 3] == 1152 + R  # clamped at the physical boundary


def test_plan_spec_example_carry():
    # S:L61 "nz=32, R=1, n=4, k=2": 2kR = 4 planes resident; with R=4 the same law is 2kR = 16
    p = oracle.plan(64, 4, 2)
    assert p[1, 5] - p[1, 4] == 2 * 2 * R
    assert p[1, 6] == p[1, 5] and p[1, 7] == p[1, 3]
    q = oracle.plan(64, 4, 2, sharing=False)
    assert q[1, 6] == q[1, 2]  # no sharing: the whole extent is transferred


@pytest.mark.parametrize("nz,n,k", [(64, 4, 2), (128, 8, 3), (48, 3, 1), (40, 3, 2), (16, 1, 3)])
def test_plan_coverage_bruteforce(nz, n, k):
    p = oracle.plan(nz, n, k)
    owned = np.zeros(nz, dtype=int)
    for i in range(n):
        owned[p[i, 0]:p[i, 1]] += 1
        assert p[i, 1] - p[i, 0] > k * R
        assert p[i, 0] % 4 == 0 and p[i, 1] % 4 == 0
    assert np.all(owned == 1)
    for i in range(n):
        ext = set(range(p[i, 2], p[i, 3]))
        body = set(range(p[i, 6], p[i, 7]))
        carry = set(range(p[i, 4], p[i, 5]))
        assert body | carry == ext and not (body & carry)
        if i > 0:
            prev_ext = set(range(p[i - 1, 2], p[i - 1, 3]))
            assert carry == prev_ext & ext  # carry is exactly what the previous chunk left on the GPU


@pytest.mark.parametrize("nz,n,k", [(8, 3, 1), (32, 4, 2), (64, 16, 1), (20, 3, 0)])
def test_plan_rejects(nz, n, k):
    with pytest.raises(oracle.OracleError):
        oracle.plan(nz, n, k)


def _stores(nx, ny, nz, codec, q, kind="layered"):
    vel, p0 = synth.fields(nx, ny, nz, kind=kind)
    return vel, p0, [oracle.encode_planes(a, codec, q) for a in (vel, p0, p0)]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_identity_pipeline_bitwise_equals_incore(n, k):
    nx, ny, nz = 12, 8, 128
    vel, p0, (Sv, Sp, Sc) = _stores(nx, ny, nz, oracle.CODEC_IDENTITY, 0)
    ax, ay = nx + 2 * R, ny + 2 * R
    dt = synth.dt_for()
    T = 2 * k
    oracle.pipeline(ax, ay, nz, n, k, dt, T, oracle.CODEC_IDENTITY, 0, Sv, Sp, Sc)
    pp, pc = oracle.incore(vel, p0.copy(), p0.copy(), dt, T)
    got_p = Sp.view(np.float32).reshape(pp.shape)
    got_c = Sc.view(np.float32).reshape(pc.shape)
    assert np.array_equal(got_c.view(np.uint32), pc.view(np.uint32))
    assert np.array_equal(got_p.view(np.uint32), pp.view(np.uint32))
    assert not np.array_equal(pc, p0)


@pytest.mark.parametrize("r", [8, 16, 24])
@pytest.mark.parametrize("n,k", [(4, 2), (3, 1), (2, 3)])
def test_lossy_pipeline_equals_incore_with_injected_roundtrip(r, n, k):
    q = r - 1
    nx, ny, nz = 16, 12, 96
    vel, p0, (Sv, Sp, Sc) = _stores(nx, ny, nz, oracle.CODEC_BLOCKQUANT, q)
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    dt = synth.dt_for()
    T = 3 * k
    oracle.pipeline(ax, ay, nz, n, k, dt, T, oracle.CODEC_BLOCKQUANT, q, Sv, Sp, Sc)
    # independent formulation: whole-field round trip, k in-core steps, round trip, ...
    rt = lambda a: oracle.decode_planes(oracle.encode_planes(a, 1, q), ax, ay, az, 1, q)
    v = rt(vel)
    pp, pc = rt(p0), rt(p0)
    for _ in range(T // k):
        pp, pc = oracle.incore(v, pp, pc, dt, k)
        pp, pc = rt(pp), rt(pc)
    got_p = oracle.decode_planes(Sp, ax, ay, az, 1, q)
    got_c = oracle.decode_planes(Sc, ax, ay, az, 1, q)
    assert np.array_equal(got_p, pp) and np.array_equal(got_c, pc)


def test_c1_lossy_error_vs_incore_is_small():
    # BASELINE configs[0]: 64^3, 4 blocks, 4 steps, k=2, rate 16
    nx = ny = nz = 64
    q = 15
    vel, p0, (Sv, Sp, Sc) = _stores(nx, ny, nz, oracle.CODEC_BLOCKQUANT, q)
    ax = ay = az = nx + 2 * R
    dt = synth.dt_for()
    oracle.pipeline(ax, ay, nz, 4, 2, dt, 4, oracle.CODEC_BLOCKQUANT, q, Sv, Sp, Sc)
    _, pc = oracle.incore(vel, p0.copy(), p0.copy(), dt, 4)
    got = oracle.decode_planes(Sc, ax, ay, az, 1, q)
    err = np.abs(got.astype(np.float64) - pc)
    rng_ = pc[R:-R, R:-R, R:-R].max() - pc[R:-R, R:-R, R:-R].min()
    rmse = np.sqrt(np.mean(err[R:-R, R:-R, R:-R] ** 2))
    psnr = 20 * np.log10(rng_ / rmse)
    assert err.max() < 1e-3 and psnr > 80.0
