"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/oracle.c header).

Thin ctypes/numpy wrapper around liboracle.so, the plain CPU implementation of
arXiv 2204.11315's out-of-core compressed stencil path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this package.  The product path (paper_2204_11315_b200/) never
imports it, and this package never imports the product.

Arrays use the allocated layout (planes, ay, ax), x fastest, float32.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

R = 4  # stencil radius (P:L190 HALO=4, P:L212 25-point)
CODEC_IDENTITY = 0
CODEC_BLOCKQUANT = 1
CODEC_ZFP = 2  # the codec parameter is the rate (bits/value) for ZFP, q = rate - 1 for BlockQuant
CODEC_TRUNC16 = 3  # fp32 -> bfloat16 RNE; the codec parameter is unused


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, f32, i32, vp = ctypes.c_int64, ctypes.c_float, ctypes.c_int, ctypes.c_void_p
        L.oracle_coeffs.argtypes = [vp]
        L.oracle_step.argtypes = [i64, i64, i64, vp, vp, vp, f32, i64, i64]
        L.oracle_incore.argtypes = [i64, i64, i64, vp, vp, vp, f32, i64]
        L.oracle_step_s.argtypes = [i32, i64, i64, i64, vp, vp, vp, f32, i64, i64]
        L.oracle_incore_s.argtypes = [i32, i64, i64, i64, vp, vp, vp, f32, i64]
        L.oracle_pipeline_s.argtypes = [i32, i64, i64, i64, i64, i64, f32, i64, i32, i32, vp, vp, vp]
        L.oracle_pipeline_s.restype = i32
        L.oracle_bq_encode_block.argtypes = [vp, i32, vp]
        L.oracle_bq_encode_block.restype = i32
        L.oracle_bq_decode_block.argtypes = [vp, i32, vp]
        L.oracle_plane_bytes.argtypes = [i64, i64, i32, i32]
        L.oracle_plane_bytes.restype = i64
        L.oracle_encode_planes.argtypes = [i64, i64, i64, vp, i32, i32, vp]
        L.oracle_encode_planes.restype = i32
        L.oracle_decode_planes.argtypes = [i64, i64, i64, vp, i32, i32, vp]
        L.oracle_plan.argtypes = [i64, i64, i64, i32, vp]
        L.oracle_plan.restype = i32
        L.oracle_pipeline.argtypes = [i64, i64, i64, i64, i64, f32, i64, i32, i32, vp, vp, vp]
        L.oracle_pipeline.restype = i32
        L.oracle_zfp_encode_block.argtypes = [vp, i32, vp]
        L.oracle_zfp_encode_block.restype = i32
        L.oracle_zfp_decode_block.argtypes = [vp, i32, vp]
        L.oracle_zfp_fwd_lift.argtypes = [vp, i32]
        L.oracle_zfp_inv_lift.argtypes = [vp, i32]
        L.oracle_zfp_fwd_xform.argtypes = [vp]
        L.oracle_zfp_inv_xform.argtypes = [vp]
        L.oracle_zfp_int2uint.argtypes = [ctypes.c_int32]
        L.oracle_zfp_int2uint.restype = ctypes.c_uint32
        L.oracle_zfp_uint2int.argtypes = [ctypes.c_uint32]
        L.oracle_zfp_uint2int.restype = ctypes.c_int32
        L.oracle_tr16_encode.argtypes = [f32]
        L.oracle_tr16_encode.restype = ctypes.c_uint16
        L.oracle_tr16_decode.argtypes = [ctypes.c_uint16]
        L.oracle_tr16_decode.restype = f32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, rc: int):
        super().__init__(f"oracle returned status {rc}")
        self.rc = rc


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's plane loops (timing only; results are thread-count independent)."""
    lib().oracle_set_threads(int(n))


def coeffs() -> np.ndarray:
    c = np.zeros(5, dtype=np.float64)
    lib().oracle_coeffs(_p(c))
    return c


STENCIL_ACOUSTIC25 = 0
STENCIL_STAR7 = 1


def step(vel, p_prev, p_curr, dt, z_lo, z_hi, stencil=STENCIL_ACOUSTIC25):
    """One leapfrog step on buffer planes [z_lo, z_hi); p_prev is overwritten with p_next."""
    planes, ay, ax = p_curr.shape
    for a in (vel, p_prev, p_curr):
        assert a.dtype == np.float32 and a.shape == (planes, ay, ax)
    lib().oracle_step_s(stencil, ax, ay, planes, _p(vel), _p(p_prev), _p(p_curr), float(dt), z_lo, z_hi)


def incore(vel, p_prev, p_curr, dt, steps, stencil=STENCIL_ACOUSTIC25):
    """T plain steps in place; returns (p_prev, p_curr) = levels (T-1, T)."""
    az, ay, ax = p_curr.shape
    lib().oracle_incore_s(stencil, ax, ay, az, _p(vel), _p(p_prev), _p(p_curr), float(dt), steps)
    return p_prev, p_curr


def encode_block(x, q: int) -> bytes:
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(64)
    rec = np.zeros(8 * (q + 1), dtype=np.uint8)
    rc = lib().oracle_bq_encode_block(_p(x), q, _p(rec))
    if rc:
        raise OracleError(rc)
    return rec.tobytes()


def decode_block(rec: bytes, q: int) -> np.ndarray:
    r = np.frombuffer(rec, dtype=np.uint8).copy()
    x = np.zeros(64, dtype=np.float32)
    lib().oracle_bq_decode_block(_p(r), q, _p(x))
    return x


def plane_bytes(ax, ay, codec, q) -> int:
    return int(lib().oracle_plane_bytes(ax, ay, codec, q))


def encode_planes(src: np.ndarray, codec: int, q: int) -> np.ndarray:
    planes, ay, ax = src.shape
    src = np.ascontiguousarray(src, dtype=np.float32)
    out = np.zeros(plane_bytes(ax, ay, codec, q) * planes, dtype=np.uint8)
    rc = lib().oracle_encode_planes(ax, ay, planes, _p(src), codec, q, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def decode_planes(buf: np.ndarray, ax, ay, planes, codec, q) -> np.ndarray:
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    out = np.zeros((planes, ay, ax), dtype=np.float32)
    lib().oracle_decode_planes(ax, ay, planes, _p(buf), codec, q, _p(out))
    return out


def plan(nz, n, k, sharing=True) -> np.ndarray:
    out = np.zeros((n, 8), dtype=np.int64)
    rc = lib().oracle_plan(nz, n, k, int(sharing), _p(out))
    if rc:
        raise OracleError(rc)
    return out


def pipeline(ax, ay, nz, n, k, dt, steps, codec, q, S_vel, S_prev, S_curr, stencil=STENCIL_ACOUSTIC25):
    """Run the method on compressed stores in place (S_prev/S_curr updated)."""
    rc = lib().oracle_pipeline_s(stencil, ax, ay, nz, n, k, float(dt), steps, codec, q,
                                 _p(S_vel), _p(S_prev), _p(S_curr))
    if rc:
        raise OracleError(rc)
    return S_prev, S_curr


# ---- ZFP (NEXT-1) ------------------------------------------------------------
def zfp_encode_block(x, rate: int) -> bytes:
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(64)
    rec = np.zeros(rate, dtype=np.uint64)
    rc = lib().oracle_zfp_encode_block(_p(x), rate, _p(rec))
    if rc:
        raise OracleError(rc)
    return rec.tobytes()


def zfp_decode_block(rec: bytes, rate: int) -> np.ndarray:
    r = np.frombuffer(rec, dtype=np.uint64).copy()
    x = np.zeros(64, dtype=np.float32)
    lib().oracle_zfp_decode_block(_p(r), rate, _p(x))
    return x


def zfp_lift(v, inverse=False):
    a = np.ascontiguousarray(v, dtype=np.int32).copy()
    (lib().oracle_zfp_inv_lift if inverse else lib().oracle_zfp_fwd_lift)(_p(a), 1)
    return a


def zfp_xform(b, inverse=False):
    a = np.ascontiguousarray(b, dtype=np.int32).reshape(64).copy()
    (lib().oracle_zfp_inv_xform if inverse else lib().oracle_zfp_fwd_xform)(_p(a))
    return a


def zfp_int2uint(x: int) -> int:
    return int(lib().oracle_zfp_int2uint(x))


def zfp_uint2int(u: int) -> int:
    return int(lib().oracle_zfp_uint2int(u))


# ---- Truncate-16 -----------------------------------------------------------------
def tr16_encode(x: float) -> int:
    return int(lib().oracle_tr16_encode(float(np.float32(x))))


def tr16_decode(h: int) -> float:
    return float(lib().oracle_tr16_decode(h))
