"""Pins for the oracle's BlockQuant / identity codec.

Pinned against: the hand-derived closed-form golden block (tests/golden/bq_ramp_q15.txt),
exhaustive bin-centre blocks for q <= 8, the error bound of uniform quantisation
 on 1e5 random blocks per rate, the fixed-rate size law (S:L191,
S:L237), monotonicity, constant blocks, rejection of non-finite data
(S:L200), identity bitwise and segment independence.
"""
import math
import os
import struct

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bq_ramp_q15.txt")
RATES = [8, 12, 16, 24]  # BASELINE configs[2] rate sweep; q = r - 1


def _golden():
    d = {}
    for line in open(GOLD):
        if line.strip() and not line.startswith("#"):
            k, v = line.split()
            d[k] = v
    return d


def _planes_of(rec, q):
    return [struct.unpack_from("<Q", rec, 8 + 8 * (q - 1 - b))[0] for b in range(q)]


def _codes_of(rec, q):
    planes = _planes_of(rec, q)
    return [sum(((planes[b] >> j) & 1) << b for b in range(q)) for j in range(64)]


def test_golden_ramp_block_q15():
    g = _golden()
    rec = oracle.encode_block(np.arange(64, dtype=np.float32), 15)
    assert len(rec) == 128
    assert rec[0:4].hex() == bytes.fromhex(g["mn_hex"])[::-1].hex()
    assert struct.unpack("<I", rec[4:8])[0] == int(g["mx_hex"], 16)
    planes = _planes_of(rec, 15)
    assert planes[14] == int(g["P14_hex"], 16)
    assert planes[0] == int(g["P0_hex"], 16)
    codes = _codes_of(rec, 15)
    assert codes == [min(520 * j + (8 * j) // 63, 32767) for j in range(64)]
    dec = oracle.decode_block(rec, 15)
    want = np.array([(c + 0.5) * 63 / 32768 for c in codes], dtype=np.float64)
    assert np.array_equal(dec.astype(np.float64), want)  # exact: <= 22 significant bits
    err = np.abs(dec.astype(np.float64) - np.arange(64))
    assert err.max() == int(g["max_abs_err_num"]) / int(g["max_abs_err_den"])
    assert err[0] == err[63] == err.max()  # both end bins sit half a step from their centre


@pytest.mark.parametrize("q", range(1, 9))
def test_bin_centres_exhaustive(q):
    # range is a power of two -> scale = 2^q/range exact; values at bin centres map to their code
    step = 2.0 ** -3
    mx = (2 ** q) * step
    codes = list(range(2 ** q))
    for i in range(0, len(codes), 62):
        chunk = codes[i:i + 62]
        chunk = chunk + [chunk[-1]] * (62 - len(chunk))
        x = np.array([0.0, mx] + [(c + 0.5) * step for c in chunk], dtype=np.float32)
        rec = oracle.encode_block(x, q)
        got = _codes_of(rec, q)
        assert got[0] == 0 and got[1] == 2 ** q - 1
        assert got[2:] == chunk
        dec = oracle.decode_block(rec, q)
        assert np.array_equal(dec[2:], x[2:])


def _blocks_to_planes(blocks):
    n = blocks.shape[0]
    b = blocks.reshape(n, 4, 4, 4)  # (block, zi, yi, xi)
    return np.ascontiguousarray(b.transpose(1, 2, 0, 3).reshape(4, 4, 4 * n))


def _planes_to_blocks(arr):
    n = arr.shape[2] // 4
    return arr.reshape(4, 4, n, 4).transpose(2, 0, 1, 3).reshape(n, 64)


@pytest.mark.parametrize("r", RATES)
def test_error_bound_1e5_random_blocks(r):
    q = r - 1
    blocks = synth.random_blocks(100_000, seed=r)
    arr = _blocks_to_planes(blocks)
    enc = oracle.encode_planes(arr, oracle.CODEC_BLOCKQUANT, q)
    assert enc.size == 100_000 * 8 * (q + 1)  # fixed-rate law
    dec = _planes_to_blocks(oracle.decode_planes(enc, arr.shape[2], 4, 4, oracle.CODEC_BLOCKQUANT, q))
    x = blocks.astype(np.float64)
    xh = dec.astype(np.float64)
    mn, mx = x.min(axis=1, keepdims=True), x.max(axis=1, keepdims=True)
    amax = np.maximum(np.abs(mn), np.abs(mx))
    ulp = np.spacing(amax.astype(np.float32)).astype(np.float64)
    bound = (mx - mn) / 2.0 ** (q + 1) + 8 * ulp + 2.0 ** -100
    assert np.all(np.abs(x - xh) <= bound)
    # decoded values stay inside [mn, mx] up to one rounding
    assert np.all(xh >= mn - ulp) and np.all(xh <= mx + ulp)
    # monotone within a block: x_i <= x_j  =>  x^_i <= x^_j
    order = np.argsort(x, axis=1, kind="stable")
    xs = np.take_along_axis(xh, order, axis=1)
    assert np.all(np.diff(xs, axis=1) >= 0)


def test_constant_signed_zero_and_subnormal_blocks():
    for val in [0.0, -0.0, 1.0, -7.25, 1e-40, 3.4e37]:
        x = np.full(64, val, dtype=np.float32)
        for q in (7, 15, 23):
            dec = oracle.decode_block(oracle.encode_block(x, q), q)
            assert np.array_equal(dec, x + np.float32(0.0)), (val, q)
            assert not np.any(np.signbit(dec)) or val < 0
    # -0 canonicalised: a block of -0 and +0 encodes like all +0
    z = np.zeros(64, dtype=np.float32)
    zm = z.copy()
    zm[::3] = -0.0
    assert oracle.encode_block(z, 15) == oracle.encode_block(zm, 15)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf, 2.0 ** 126, -(2.0 ** 127)])
def test_rejects_nonfinite_and_huge(bad):
    x = np.ones(64, dtype=np.float32)
    x[5] = bad
    with pytest.raises(oracle.OracleError) as e:
        oracle.encode_block(x, 15)
    assert e.value.rc == 6


def test_identity_codec_bitwise_and_segment_independence():
    rng = np.random.default_rng(9)
    arr = rng.normal(size=(12, 8, 12)).astype(np.float32)
    arr[0, 0, 0] = -0.0
    enc = oracle.encode_planes(arr, oracle.CODEC_IDENTITY, 0)
    assert enc.tobytes() == arr.tobytes()
    assert np.array_equal(oracle.decode_planes(enc, 12, 8, 12, oracle.CODEC_IDENTITY, 0).view(np.uint32),
                          arr.view(np.uint32))
    # BlockQuant: encoding planes [0,12) at once == encoding [0,4), [4,12) separately (independent
    # fixed-rate slabs, "compress the overlapped area ... separately")
    q = 11
    whole = oracle.encode_planes(arr, oracle.CODEC_BLOCKQUANT, q)
    parts = np.concatenate([oracle.encode_planes(arr[:4], oracle.CODEC_BLOCKQUANT, q),
                            oracle.encode_planes(arr[4:], oracle.CODEC_BLOCKQUANT, q)])
    assert np.array_equal(whole, parts)
    pb = oracle.plane_bytes(12, 8, oracle.CODEC_BLOCKQUANT, q)
    assert pb == 3 * 2 * 8 * 12 // 4
    sub = oracle.decode_planes(whole[4 * pb:8 * pb], 12, 8, 4, oracle.CODEC_BLOCKQUANT, q)
    full = oracle.decode_planes(whole, 12, 8, 12, oracle.CODEC_BLOCKQUANT, q)
    assert np.array_equal(sub, full[4:8])
