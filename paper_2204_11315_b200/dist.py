"""Multi-GPU plumbing: hand every rank's exchange-region handle to its z-slab neighbours.

The halo exchange itself runs inside the library (include/oocs.h, "multi-GPU"): an edge chunk's
encoded kR planes are stored straight into the neighbour's HBM ghost slot over NVLink (CUDA IPC peer
memory) and signalled with stream memory operations.  This module only moves the opaque
PEER_HANDLE_BYTES blobs between processes once, at set-up: torch.distributed.all_gather_object over
whatever process group is initialised (NCCL or gloo).  It never sees a halo byte.
"""
from __future__ import annotations

import torch.distributed as dist


def neighbours(handles, rank: int):
    """(lower, upper) handles of `rank` from the rank-ordered list of every rank's handle."""
    world = len(handles)
    return (handles[rank - 1] if rank > 0 else None), (handles[rank + 1] if rank + 1 < world else None)


def connect(plan, group=None, gloo: bool = False):
    """Collective over `group`: every rank publishes its plan's handle and maps its neighbours'.
    (`gloo` is accepted for call-site symmetry: the handles are host bytes on any backend.)"""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    assert plan.cfg.world == world and plan.cfg.rank == rank, "plan rank/world differ from the process group"
    handles = [None] * world
    dist.all_gather_object(handles, plan.peer_handle(), group=group)
    lower, upper = neighbours(handles, rank)
    plan.peer_connect(lower, upper)
    dist.barrier(group)


def connect_local(plans):
    """Ranks that live in one process (e.g. W plans sharing one GPU, driven from W threads): the same
    handles, exchanged in memory.  plans[r] must be rank r."""
    handles = [p.peer_handle() for p in plans]
    for r, p in enumerate(plans):
        p.peer_connect(*neighbours(handles, r))
