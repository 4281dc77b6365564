"""The set-up protocol of paper_2204_11315_b200.dist over real torch.distributed process groups (gloo,
world 2 and 4, CPU): every rank publishes its plan's exchange-region handle and must be connected with
exactly its z-slab neighbours' handles (rank-1 below, rank+1 above, none at the domain edges) -- the
halo bytes themselves then move GPU to GPU inside the library.  And the slab/ghost geometry the library
reports (oocs_plan_table) must make a rank's ghost planes coincide with its neighbours' edge planes."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

R = 4


class _StubPlan:
    """Stands in for oocs.Plan on a CPU box: a recognisable handle, records what connect() passes."""

    class _Cfg:
        def __init__(self, rank, world):
            self.rank, self.world = rank, world

    def __init__(self, rank, world):
        self.cfg = self._Cfg(rank, world)
        self.connected = None

    def peer_handle(self):
        return bytes([self.cfg.rank + 1]) * 256

    def peer_connect(self, lower, upper):
        self.connected = (lower, upper)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_11315_b200.dist import connect

        pl = _StubPlan(rank, world)
        connect(pl)
        lo, up = pl.connected
        ok = (lo == (bytes([rank]) * 256 if rank > 0 else None)) and \
             (up == (bytes([rank + 2]) * 256 if rank + 1 < world else None))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_connect_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in ps]
    [p.join(timeout=120) for p in ps]
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert [r[1] for r in res] == [True] * world


def test_local_connect_pairs_neighbours():
    from paper_2204_11315_b200.dist import connect_local

    plans = [_StubPlan(r, 3) for r in range(3)]
    connect_local(plans)
    h = [p.peer_handle() for p in plans]
    assert [p.connected for p in plans] == [(None, h[1]), (h[0], h[2]), (h[1], None)]


@pytest.mark.parametrize("world,n,k", [(2, 8, 2), (4, 8, 3), (8, 16, 4)])
def test_slab_ghost_geometry(world, n, k):
    import paper_2204_11315_b200 as oocs

    nz = 32 * n
    cfgs = [oocs.make_config(nx=16, ny=16, nz=nz, dt=0.1, n_blocks=n, tb_depth=k, rank=r, world=world)
            for r in range(world)]
    table = oocs.oocs_plan_table(cfgs[0])
    per = n // world
    slabs = [(table[r * per][0], table[(r + 1) * per - 1][1]) for r in range(world)]
    assert slabs[0][0] == 0 and slabs[-1][1] == nz
    for r in range(world - 1):
        assert slabs[r][1] == slabs[r + 1][0]
        # what rank r needs above its slab (ghost hi) is exactly what rank r+1 sends down: kR planes
        ext_last = table[(r + 1) * per - 1][3]
        assert ext_last - slabs[r][1] == k * R
        ext_first = table[(r + 1) * per][2]
        assert slabs[r + 1][0] - ext_first == k * R
