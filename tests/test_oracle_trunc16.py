"""Pins for the oracle's Truncate-16 codec (SURVEY.md §8(b) codec enum, §8(c) C-3: fp32 -> bfloat16
with round-to-nearest-even, NaN -> quiet NaN).

Pinned against: the worked tie cases of SURVEY §8(c) (tests/golden/tr16_ties.txt), the library
routine that defines the same conversion (torch's CPU fp32 -> bfloat16 cast) on every exponent and on
a million random bit patterns, the exact decode (bf16 is the upper half of binary32), the half-ulp
error bound, the fixed-rate size law and plane-range independence, and the lossy out-of-core pipeline
equal to in-core steps with an injected whole-field round trip after every sweep.
"""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
C = oracle.CODEC_TRUNC16
GOLD = os.path.join(os.path.dirname(__file__), "golden", "tr16_ties.txt")


def _enc_bits(bits: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(bits, dtype=np.uint32).view(np.float32).reshape(1, 1, -1)
    return oracle.encode_planes(x, C, 0).view(np.uint16)


def _torch_bits(bits: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(bits, dtype=np.uint32).view(np.float32).copy())
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def test_golden_tie_cases():
    rows = [l.split()[:2] for l in open(GOLD) if l.strip() and not l.startswith("#")]
    assert len(rows) == 13
    src = np.array([int(a, 16) for a, _ in rows], dtype=np.uint32)
    want = np.array([int(b, 16) for _, b in rows], dtype=np.uint16)
    got = _enc_bits(np.concatenate([src, np.zeros(3, np.uint32)]))[:13]  # ax multiple of 4
    assert np.array_equal(got, want), [(hex(a), hex(g), hex(w)) for a, g, w in zip(src, got, want) if g != w]
    for s, w in zip(src, want):
        assert oracle.tr16_encode(np.uint32(s).view(np.float32)) == w or np.isnan(np.uint32(s).view(np.float32))


def test_equals_torch_bfloat16_cast():
    rng = np.random.default_rng(11315)
    bits = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    # every exponent, with fraction patterns at and around the rounding boundary
    e = np.arange(256, dtype=np.uint32) << 23
    fr = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0x17FFF, 0x18000, 0x18001, 0x7FFFFF, 0x7F8000], np.uint32)
    grid = (e[:, None] | fr[None, :]).ravel()
    bits = np.concatenate([bits, grid, grid | 0x80000000])
    bits = bits[: bits.size // 4 * 4]
    got, want = _enc_bits(bits), _torch_bits(bits)
    isnan = np.isnan(bits.view(np.float32))
    assert np.array_equal(got[~isnan], want[~isnan])
    assert np.all(got[isnan] == 0x7FC0) and np.all((want[isnan] & 0x7FC0) == 0x7FC0)


def test_decode_exact_and_error_bound():
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(8, 12, 16)) * 10.0 ** rng.integers(-30, 30, size=(8, 12, 16))).astype(np.float32)
    enc = oracle.encode_planes(x, C, 0)
    assert enc.size == x.size * 2 == oracle.plane_bytes(16, 12, C, 0) * 8  # fixed-rate law, rate 16
    dec = oracle.decode_planes(enc, 16, 12, 8, C, 0)
    # decode = the 16 encoded bits followed by 16 zero bits (exact)
    assert np.array_equal(dec.view(np.uint32), enc.view(np.uint16).astype(np.uint32).reshape(x.shape) << 16)
    # round to nearest: |x - x^| <= half an ulp of bf16 (2^-8 relative to the leading power of two)
    lead = 2.0 ** np.floor(np.log2(np.abs(x.astype(np.float64))))
    assert np.all(np.abs(dec.astype(np.float64) - x) <= lead * 2.0**-8)
    # plane-range independence: encoding planes [0,4) and [4,8) separately gives the same bytes
    assert np.array_equal(enc, np.concatenate([oracle.encode_planes(x[:4], C, 0), oracle.encode_planes(x[4:], C, 0)]))


@pytest.mark.parametrize("n,k", [(4, 2), (3, 1)])
def test_trunc16_pipeline_equals_incore_with_injected_roundtrip(n, k):
    R = oracle.R
    nx, ny, nz = 16, 12, 96
    vel, p0 = synth.fields(nx, ny, nz)
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    Sv, Sp, Sc = [oracle.encode_planes(a, C, 0) for a in (vel, p0, p0)]
    dt = synth.dt_for()
    T = 3 * k
    oracle.pipeline(ax, ay, nz, n, k, dt, T, C, 0, Sv, Sp, Sc)
    rt = lambda a: oracle.decode_planes(oracle.encode_planes(a, C, 0), ax, ay, az, C, 0)
    v = rt(vel)
    pp, pc = rt(p0), rt(p0)
    for _ in range(T // k):
        pp, pc = oracle.incore(v, pp, pc, dt, k)
        pp, pc = rt(pp), rt(pc)
    assert np.array_equal(oracle.decode_planes(Sp, ax, ay, az, C, 0), pp)
    assert np.array_equal(oracle.decode_planes(Sc, ax, ay, az, C, 0), pc)
