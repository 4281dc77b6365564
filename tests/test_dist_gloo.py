"""The halo-exchange protocol of paper_2204_11315_b200.dist over real torch.distributed process groups
(gloo, world 2 and 4, CPU): every rank's receive buffers must hold exactly its neighbours' send
buffers, and the slab/ghost geometry the library reports (oocs_plan_table) must make a rank's ghost
planes coincide with its neighbours' edge planes."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

R = 4


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_11315_b200.dist import halo_exchange

        n = 1000 + rank
        send_lo = torch.full((64,), 10 * rank + 1, dtype=torch.uint8)
        send_hi = torch.full((64,), 10 * rank + 2, dtype=torch.uint8)
        recv_lo = torch.zeros(64, dtype=torch.uint8)
        recv_hi = torch.zeros(64, dtype=torch.uint8)
        halo_exchange(send_lo, send_hi, recv_lo, recv_hi, rank, world)
        ok = True
        if rank > 0:
            ok &= bool(torch.all(recv_lo == 10 * (rank - 1) + 2))
        if rank + 1 < world:
            ok &= bool(torch.all(recv_hi == 10 * (rank + 1) + 1))
        q.put((rank, ok, n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_halo_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 100
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in ps]
    [p.join(timeout=120) for p in ps]
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert [r[1] for r in res] == [True] * world


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
