"""paper_2204_11315_b200 — B200-native out-of-core compressed stencil (arXiv 2204.11315).

Thin ctypes binding over the C ABI in include/oocs.h (liboocs.so, built
in-tree for sm_100a by _build.py).  Argument marshalling only: every step of
the hot path runs inside the library's CUDA kernels and streams.  There is no
CPU fallback: importing works on a CPU-only box (for the host-only planning
calls), but every GPU call fails loudly if the extension or the GPU is
missing.

Function names mirror the C ABI (oocs_plan_create, oocs_run, ...); the
``Plan`` class is a convenience wrapper over the same calls.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "R", "OOCS_OK", "OocsError", "Config", "Stats", "PlanInfo", "Block", "Op",
    "lib", "oocs_plan_table", "oocs_schedule", "oocs_encoded_bytes", "oocs_plan_create",
    "oocs_plan_query", "oocs_plan_estimate", "oocs_destroy", "oocs_load", "oocs_store", "oocs_load_device", "oocs_store_device", "oocs_store_read_raw",
    "oocs_store_write_raw", "oocs_run", "oocs_run_async", "oocs_wait", "oocs_decode", "oocs_encode", "oocs_step",
    "oocs_peer_handle", "oocs_peer_connect", "PEER_HANDLE_BYTES", "Plan", "XOFF", "pitch_for",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OOCS_LIB", os.path.join(HERE, "liboocs.so"))  # override: experiments only
R = 4
XOFF = 32 - R

OOCS_OK = 0
STATUS = {0: "OK", 2: "CONFIG", 3: "DEVICE_OOM", 4: "VERIFY", 5: "IO", 6: "DATA", 7: "HOST_OOM",
          8: "CUDA", 9: "EXCHANGE", 10: "STATE"}
CODEC = {"identity": 0, "blockquant": 1, "zfp": 2, "trunc16": 3}
MODE = {"baseline": 0, "compress": 1, "swb": 2, "dwb": 3}
STORE = {"host": 0, "device": 1}
SCHED = {"alg1": 0, "dag": 1, "dag_func": 2}
STENCIL = {"acoustic25": 0, "star7": 1}
FLAG_PROFILE = 1
FLAG_RESIDENT_VELOCITY = 2
FLAG_TIMELINE = 8
FLAG_LANE_SINGLE_STREAM = 16
FLAG_LANE_SPLIT_STREAMS = 32
FLAG_DECODED_VELOCITY = 64
FLAG_FUSE_DECODE = 128
EXECUTOR = {"dispatch": 0, "single": FLAG_LANE_SINGLE_STREAM, "split": FLAG_LANE_SPLIT_STREAMS}
OP_KINDS = ["H2D", "CARRY", "DECODE", "STEP", "ENCODE", "D2H", "RECORD", "WAIT", "SEND"]
PEER_HANDLE_BYTES = 256
EV_KINDS = ["H2D", "DEC", "ENC", "D2H", "CARRY", "NODE"]

i32, i64, u32, u64, f32, f64, vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_float, ctypes.c_double, ctypes.c_void_p)


class Config(ctypes.Structure):
    _fields_ = [("struct_size", u32), ("nx", i64), ("ny", i64), ("nz", i64), ("dt", f32),
                ("n_blocks", i32), ("tb_depth", i32), ("codec", i32), ("rate_bits", i32), ("mode", i32),
                ("region_sharing", i32), ("n_lanes", i32), ("schedule", i32), ("store", i32), ("device", i32), ("rank", i32), ("world", i32),
                ("flags", u32), ("device_capacity", u64),
                # ABI 2
                ("stencil", i32), ("v_max", f32), ("ext_streams", vp * 8)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("ax", i64), ("ay", i64), ("az", i64), ("pitch", i64), ("plane_bytes", i64), ("z_lo", i64),
                ("z_hi", i64), ("store_lo", i64), ("store_hi", i64), ("block_lo", i32), ("block_hi", i32),
                ("max_ext_planes", i64), ("arena_bytes", u64), ("working_set_bytes", u64),
                ("staging_bytes", u64), ("store_bytes", u64), ("n_working_sets", i32), ("n_lanes", i32)]


class Stats(ctypes.Structure):
    _fields_ = [("wall_ms", f64), ("kernel_ms", f64 * 3), ("kernel_launches", i64 * 3), ("bytes_h2d", u64),
                ("bytes_d2h", u64), ("bytes_d2d", u64), ("bytes_exchange", u64), ("cell_updates", u64),
                ("cell_updates_computed", u64), ("alg_bytes", u64 * 3), ("data_error", i32), ("copy_launches", i32),
                ("busy_ms", f64 * 4)]

    def as_dict(self):
        return {
            "wall_ms": self.wall_ms, "kernel_ms": list(self.kernel_ms),
            "kernel_launches": list(self.kernel_launches), "bytes_h2d": self.bytes_h2d,
            "bytes_d2h": self.bytes_d2h, "bytes_d2d": self.bytes_d2d, "bytes_exchange": self.bytes_exchange,
            "cell_updates": self.cell_updates, "cell_updates_computed": self.cell_updates_computed,
            "alg_bytes": list(self.alg_bytes), "data_error": self.data_error,
        }


class Block(ctypes.Structure):
    _fields_ = [("own_lo", i64), ("own_hi", i64), ("ext_lo", i64), ("ext_hi", i64), ("carry_lo", i64),
                ("carry_hi", i64), ("body_lo", i64), ("body_hi", i64)]


class Op(ctypes.Structure):
    _fields_ = [("kind", i32), ("lane", i32), ("g", i64), ("block", i32), ("sweep", i32), ("arg", i32),
                ("pad", i32), ("ev_g", i64)]


class Span(ctypes.Structure):
    _fields_ = [("kind", i32), ("lane", i32), ("g", i64), ("block", i32), ("sweep", i32), ("arg", i32),
                ("pad", i32), ("start_ms", f64), ("end_ms", f64), ("host_ms", f64)]


class OocsError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: OOCS_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load liboocs.so (never falls back to anything else)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        sig = {
            "oocs_plan_table": ([P(Config), vp], i32),
            "oocs_schedule": ([P(Config), i64, vp, i64, P(i64)], i32),
            "oocs_encoded_bytes": ([P(Config), i64, P(u64)], i32),
            "oocs_plan_create": ([P(Config), P(vp)], i32),
            "oocs_plan_create_in": ([P(Config), vp, u64, P(vp)], i32),
            "oocs_plan_query": ([vp, P(PlanInfo)], i32),
            "oocs_plan_estimate": ([P(Config), P(PlanInfo)], i32),
            "oocs_peer_handle": ([vp, vp], i32),
            "oocs_peer_connect": ([vp, vp, vp], i32),
            "oocs_destroy": ([vp], i32),
            "oocs_load": ([vp, i32, vp, i64, i64], i32),
            "oocs_load_device": ([vp, i32, vp, i64, i64], i32),
            "oocs_store_device": ([vp, i32, vp, i64, i64], i32),
            "oocs_store": ([vp, i32, vp, i64, i64], i32),
            "oocs_store_read_raw": ([vp, i32, vp, i64, i64], i32),
            "oocs_store_write_raw": ([vp, i32, vp, i64, i64], i32),
            "oocs_run": ([vp, i64, P(Stats)], i32),
            "oocs_run_async": ([vp, i64], i32),
            "oocs_wait": ([vp, vp, i64, P(i64)], i32),
            "oocs_schedule_at": ([P(Config), i64, i64, vp, i64, P(i64)], i32),
            "oocs_timeline": ([vp, vp, i64, P(i64)], i32),
            "oocs_decode": ([vp, vp, i64, i64, i64, i64, i32, i32, vp], i32),
            "oocs_encode": ([vp, vp, i64, i64, i64, i64, i32, i32, vp, vp], i32),
            "oocs_step": ([vp, vp, vp, i64, i64, i64, i64, f32, i64, i64, i32, vp], i32),
            "oocs_last_error": ([], ctypes.c_char_p),
            "oocs_abi_version": ([], i32),
            "oocs_abi_sizes": ([vp], None),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != OOCS_OK:
        raise OocsError(st, where, lib().oocs_last_error().decode())


def make_config(nx, ny, nz, dt, n_blocks, tb_depth, codec="blockquant", rate_bits=16, mode="swb",
                region_sharing=True, store="host", device=0, rank=0, world=1, profile=False,
                device_capacity=0, n_lanes=0, resident_velocity=False, schedule="alg1",
                timeline=False, executor="dispatch", decoded_velocity=False, stencil="acoustic25", v_max=0.0,
                ext_streams=(), fuse_decode=False) -> Config:
    """ext_streams: up to 8 integer cudaStream_t handles (e.g. torch.cuda.Stream().cuda_stream), lane order."""
    c = Config()
    c.struct_size = ctypes.sizeof(Config)
    c.nx, c.ny, c.nz = nx, ny, nz
    c.dt = float(dt)
    c.n_blocks, c.tb_depth = n_blocks, tb_depth
    c.codec = CODEC[codec] if isinstance(codec, str) else codec
    c.rate_bits = rate_bits
    c.mode = MODE[mode] if isinstance(mode, str) else mode
    c.region_sharing = int(region_sharing)
    c.n_lanes = n_lanes
    c.schedule = SCHED[schedule] if isinstance(schedule, str) else schedule
    c.store = STORE[store] if isinstance(store, str) else store
    c.device, c.rank, c.world = device, rank, world
    c.flags = ((FLAG_PROFILE if profile else 0) | (FLAG_RESIDENT_VELOCITY if resident_velocity else 0)
               | (FLAG_TIMELINE if timeline else 0) | EXECUTOR[executor]
               | (FLAG_DECODED_VELOCITY if decoded_velocity else 0) | (FLAG_FUSE_DECODE if fuse_decode else 0))
    c.device_capacity = device_capacity
    c.stencil = STENCIL[stencil] if isinstance(stencil, str) else stencil
    c.v_max = float(v_max)
    assert len(ext_streams) <= 8
    for i, h in enumerate(ext_streams):
        c.ext_streams[i] = h or None
    return c


def pitch_for(ax: int) -> int:
    return (XOFF + ax + 31) // 32 * 32


# ---- host-only calls --------------------------------------------------------
def oocs_plan_table(cfg: Config):
    out = (Block * cfg.n_blocks)()
    _check(lib().oocs_plan_table(ctypes.byref(cfg), out), "oocs_plan_table")
    return [(b.own_lo, b.own_hi, b.ext_lo, b.ext_hi, b.carry_lo, b.carry_hi, b.body_lo, b.body_hi) for b in out]


def oocs_schedule(cfg: Config, steps: int, first_sweep: int = 0):
    """The lowered op list of a run of `steps` steps (oocs_schedule_at: after `first_sweep` sweeps)."""
    n = i64(0)
    _check(lib().oocs_schedule_at(ctypes.byref(cfg), steps, first_sweep, None, 0, ctypes.byref(n)), "oocs_schedule")
    arr = (Op * n.value)()
    _check(lib().oocs_schedule_at(ctypes.byref(cfg), steps, first_sweep, arr, n.value, ctypes.byref(n)),
           "oocs_schedule")
    return [dict(kind=OP_KINDS[o.kind], lane=o.lane, g=o.g, block=o.block, sweep=o.sweep, arg=o.arg,
                 ev=(EV_KINDS[o.arg] if o.kind in (6, 7) else None), ev_g=o.ev_g) for o in arr]


def oocs_plan_estimate(cfg: Config) -> PlanInfo:
    info = PlanInfo()
    _check(lib().oocs_plan_estimate(ctypes.byref(cfg), ctypes.byref(info)), "oocs_plan_estimate")
    return info


def oocs_encoded_bytes(cfg: Config, planes: int) -> int:
    b = u64(0)
    _check(lib().oocs_encoded_bytes(ctypes.byref(cfg), planes, ctypes.byref(b)), "oocs_encoded_bytes")
    return b.value


# ---- plan lifetime / state ---------------------------------------------------
def oocs_plan_create(cfg: Config):
    h = vp()
    _check(lib().oocs_plan_create(ctypes.byref(cfg), ctypes.byref(h)), "oocs_plan_create")
    return h


def oocs_plan_create_in(cfg: Config, arena_ptr: int, arena_bytes: int):
    h = vp()
    _check(lib().oocs_plan_create_in(ctypes.byref(cfg), arena_ptr, arena_bytes, ctypes.byref(h)),
           "oocs_plan_create_in")
    return h


def oocs_plan_query(h) -> PlanInfo:
    info = PlanInfo()
    _check(lib().oocs_plan_query(h, ctypes.byref(info)), "oocs_plan_query")
    return info


def oocs_destroy(h):
    lib().oocs_destroy(h)


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(vp)


def oocs_load(h, array: int, src: np.ndarray, a_lo: int, a_hi: int):
    src = np.ascontiguousarray(src, dtype=np.float32)
    _check(lib().oocs_load(h, array, _ptr(src), a_lo, a_hi), "oocs_load")


def oocs_load_device(h, array: int, src_ptr: int, a_lo: int, a_hi: int):
    """src_ptr: DEVICE pointer to (a_hi-a_lo, ay, ax) float32 on the plan's device."""
    _check(lib().oocs_load_device(h, array, src_ptr, a_lo, a_hi), "oocs_load_device")


def oocs_store_device(h, array: int, dst_ptr: int, a_lo: int, a_hi: int):
    """dst_ptr: DEVICE pointer to (a_hi-a_lo, ay, ax) float32 on the plan's device."""
    _check(lib().oocs_store_device(h, array, dst_ptr, a_lo, a_hi), "oocs_store_device")


def oocs_store(h, array: int, dst: np.ndarray, a_lo: int, a_hi: int):
    assert dst.dtype == np.float32
    _check(lib().oocs_store(h, array, _ptr(dst), a_lo, a_hi), "oocs_store")


def oocs_store_read_raw(h, array: int, dst: np.ndarray, a_lo: int, a_hi: int):
    _check(lib().oocs_store_read_raw(h, array, _ptr(dst), a_lo, a_hi), "oocs_store_read_raw")


def oocs_store_write_raw(h, array: int, src: np.ndarray, a_lo: int, a_hi: int):
    src = np.ascontiguousarray(src)
    _check(lib().oocs_store_write_raw(h, array, _ptr(src), a_lo, a_hi), "oocs_store_write_raw")


def oocs_run(h, steps: int) -> Stats:
    st = Stats()
    _check(lib().oocs_run(h, steps, ctypes.byref(st)), "oocs_run")
    return st


def oocs_run_async(h, steps: int):
    _check(lib().oocs_run_async(h, steps), "oocs_run_async")


def oocs_wait(h) -> list:
    """Complete every run in flight; their Stats in issue order."""
    n = i64(0)
    cap = 64
    arr = (Stats * cap)()
    _check(lib().oocs_wait(h, arr, cap, ctypes.byref(n)), "oocs_wait")
    return [arr[i] for i in range(min(n.value, cap))]


def oocs_timeline(h):
    """Spans of the last run (OOCS_FLAG_TIMELINE) as dicts, in schedule order."""
    n = i64(0)
    _check(lib().oocs_timeline(h, None, 0, ctypes.byref(n)), "oocs_timeline")
    arr = (Span * n.value)()
    _check(lib().oocs_timeline(h, arr, n.value, ctypes.byref(n)), "oocs_timeline")
    return [dict(kind=OP_KINDS[s.kind], lane=s.lane, g=s.g, block=s.block, sweep=s.sweep, arg=s.arg,
                 start_ms=s.start_ms, end_ms=s.end_ms, host_ms=s.host_ms) for s in arr]


def oocs_peer_handle(h) -> bytes:
    """This rank's exchange-region handle (multi-GPU, world > 1): PEER_HANDLE_BYTES opaque bytes."""
    buf = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
    _check(lib().oocs_peer_handle(h, buf), "oocs_peer_handle")
    return buf.raw


def oocs_peer_connect(h, lower: bytes | None, upper: bytes | None):
    """Map rank-1's (lower) and rank+1's (upper) exchange regions; None at the domain edges."""
    lo = ctypes.create_string_buffer(lower, PEER_HANDLE_BYTES) if lower is not None else None
    up = ctypes.create_string_buffer(upper, PEER_HANDLE_BYTES) if upper is not None else None
    _check(lib().oocs_peer_connect(h, lo, up), "oocs_peer_connect")


# ---- kernel-level calls on caller device memory (integer device pointers) ---------
def oocs_decode(src_ptr: int, dst_ptr: int, ax, ay, planes, pitch, codec, rate_bits, stream=0):
    _check(lib().oocs_decode(src_ptr, dst_ptr, ax, ay, planes, pitch, codec, rate_bits, stream or None),
           "oocs_decode")


def oocs_encode(src_ptr: int, dst_ptr: int, ax, ay, planes, pitch, codec, rate_bits, err_ptr=0, stream=0):
    _check(lib().oocs_encode(src_ptr, dst_ptr, ax, ay, planes, pitch, codec, rate_bits, err_ptr or None,
                             stream or None), "oocs_encode")


def oocs_step(vel_ptr: int, pprev_ptr: int, pcurr_ptr: int, ax, ay, planes, pitch, dt, z_lo, z_hi, stream=0, *,
              stencil="acoustic25"):
    st = STENCIL[stencil] if isinstance(stencil, str) else stencil
    _check(lib().oocs_step(vel_ptr, pprev_ptr, pcurr_ptr, ax, ay, planes, pitch, float(dt), z_lo, z_hi, st,
                           stream or None), "oocs_step")


@dataclass
class Plan:
    """Convenience owner of an oocs_plan handle (same calls as the C ABI)."""
    cfg: Config
    handle: object = None
    arena: object = None  # optional caller-owned device buffer (e.g. a torch uint8 tensor) to carve from

    def __post_init__(self):
        if self.arena is not None:
            self.handle = oocs_plan_create_in(self.cfg, self.arena.data_ptr(), self.arena.numel() * self.arena.element_size())
        else:
            self.handle = oocs_plan_create(self.cfg)
        self.info = oocs_plan_query(self.handle)

    def load(self, array, src, a_lo, a_hi):
        oocs_load(self.handle, array, src, a_lo, a_hi)

    def load_device(self, array, tensor, a_lo, a_hi):
        """tensor: contiguous float32 CUDA tensor (a_hi-a_lo, ay, ax) on the plan's device."""
        assert tensor.is_cuda and tensor.is_contiguous() and tuple(tensor.shape) == (a_hi - a_lo, self.info.ay, self.info.ax)
        import torch

        torch.cuda.current_stream(tensor.device).synchronize()  # the library reads on its own streams
        oocs_load_device(self.handle, array, tensor.data_ptr(), a_lo, a_hi)

    def store_device(self, array, tensor, a_lo, a_hi):
        assert tensor.is_cuda and tensor.is_contiguous() and tuple(tensor.shape) == (a_hi - a_lo, self.info.ay, self.info.ax)
        oocs_store_device(self.handle, array, tensor.data_ptr(), a_lo, a_hi)

    def store(self, array, a_lo, a_hi):
        out = np.empty((a_hi - a_lo, self.info.ay, self.info.ax), dtype=np.float32)
        oocs_store(self.handle, array, out, a_lo, a_hi)
        return out

    def read_raw(self, array, a_lo, a_hi):
        out = np.empty((a_hi - a_lo) * self.info.plane_bytes, dtype=np.uint8)
        oocs_store_read_raw(self.handle, array, out, a_lo, a_hi)
        return out

    def write_raw(self, array, src, a_lo, a_hi):
        oocs_store_write_raw(self.handle, array, src, a_lo, a_hi)

    def run(self, steps) -> Stats:
        return oocs_run(self.handle, steps)

    def run_async(self, steps):
        oocs_run_async(self.handle, steps)

    def wait(self) -> list:
        return oocs_wait(self.handle)

    def timeline(self):
        return oocs_timeline(self.handle)

    def peer_handle(self) -> bytes:
        return oocs_peer_handle(self.handle)

    def peer_connect(self, lower, upper):
        oocs_peer_connect(self.handle, lower, upper)

    def close(self):
        if self.handle is not None:
            oocs_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
