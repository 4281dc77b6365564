"""Multi-GPU plumbing: z-slab halo exchange over torch.distributed (NCCL on GPUs, gloo on CPU tests).

The library calls back after each sweep with device pointers to the k*R compressed
planes (x 2 pressure arrays) it must send to rank-1 / rank+1 and the buffers that
receive the neighbours' planes (include/oocs.h, oocs_exchange_fn).  This module
only moves those bytes (P2P, no collective): it never looks at their content.
"""
from __future__ import annotations

import threading

import torch
import torch.distributed as dist


class _DevPtr:
    """Zero-copy view of a raw device allocation for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_bytes(ptr: int, nbytes: int) -> torch.Tensor:
    return torch.as_tensor(_DevPtr(ptr, nbytes), device="cuda")


def halo_exchange(send_lo, send_hi, recv_lo, recv_hi, rank: int, world: int, group=None):
    """Send send_lo to rank-1 and send_hi to rank+1; receive recv_lo from rank-1, recv_hi from rank+1.
    Any of the four may be None at the domain edge.  Blocks until complete."""
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, send_lo, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_lo, rank - 1, group))
    if rank + 1 < world:
        ops.append(dist.P2POp(dist.isend, send_hi, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_hi, rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def nccl_exchange_fn(rank: int, world: int):
    """Callback for Plan.set_exchange() under torch.distributed (NCCL)."""

    def fn(sweep, sl, sh, rl, rh, nbytes, stream):
        t = lambda p: device_bytes(p, nbytes) if p else None
        halo_exchange(t(sl), t(sh), t(rl), t(rh), rank, world)
        torch.cuda.synchronize()
        return 0

    return fn


def gloo_exchange_fn(rank: int, world: int):
    """Callback for a gloo process group (testing the multi-rank path where NCCL cannot run, e.g. several
    ranks sharing one GPU): device buffers are staged through host tensors."""

    def fn(sweep, sl, sh, rl, rh, nbytes, stream):
        torch.cuda.synchronize()
        t = lambda p: device_bytes(p, nbytes).cpu() if p else None
        send_lo, send_hi = t(sl), t(sh)
        recv_lo = torch.empty(nbytes, dtype=torch.uint8) if rl else None
        recv_hi = torch.empty(nbytes, dtype=torch.uint8) if rh else None
        halo_exchange(send_lo, send_hi, recv_lo, recv_hi, rank, world)
        if rl:
            device_bytes(rl, nbytes).copy_(recv_lo)
        if rh:
            device_bytes(rh, nbytes).copy_(recv_hi)
        torch.cuda.synchronize()
        return 0

    return fn


class LoopbackExchange:
    """In-process exchange between plans of one job that share a GPU (threads, one per rank).

    Stands in for NCCL when a single GPU hosts every rank (tests): each rank posts its send
    buffers, waits for all ranks, then copies the neighbours' sends into its receive buffers."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.posted = [None] * world

    def fn(self, rank: int):
        def cb(sweep, sl, sh, rl, rh, nbytes, stream):
            self.posted[rank] = (sl, sh, nbytes)
            self.barrier.wait()
            if rank > 0:
                _, hi_of_lower, n = self.posted[rank - 1]
                device_bytes(rl, n).copy_(device_bytes(hi_of_lower, n))
            if rank + 1 < self.world:
                lo_of_upper, _, n = self.posted[rank + 1]
                device_bytes(rh, n).copy_(device_bytes(lo_of_upper, n))
            torch.cuda.synchronize()
            self.barrier.wait()  # nobody reuses its send buffers before every copy is done
            return 0

        return cb
