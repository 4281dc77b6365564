"""Decode -> first step fusion (OOCS_FLAG_FUSE_DECODE): the first step of every chunk
reads p_{t-1} (and the velocity, unless it is kept decoded) from its BlockQuant records inside the
stencil kernel.  The values are the decode kernel's
(same transpose, same IEEE operations), so every configuration must be bitwise equal to the unfused run,
which the other GPU tests tie to the oracle.  p_{t-1} is loaded with its own random halo (different from
p_t's), so a missing ring / boundary-slab decode of p_{t-1} changes the result.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def fields(nx, ny, nz):
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(7)
    # p_{t-1}: p_t plus a perturbation everywhere, the halo included
    pm = (p0 + 1e-3 * rng.standard_normal(p0.shape)).astype(np.float32)
    return vel, pm, p0


def run(nx, ny, nz, n, k, steps, fuse, rate=16, mode="swb", store="host", split=None, **kw):
    vel, pm, p0 = fields(nx, ny, nz)
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, rate_bits=rate,
                         mode=mode, store=store, fuse_decode=fuse, **kw)
    pl = oocs.Plan(c)
    az = nz + 2 * R
    pl.load(0, vel, 0, az)
    pl.load(1, pm, 0, az)
    pl.load(2, p0, 0, az)
    for s in (split or [steps]):
        pl.run(s)
    out = (pl.read_raw(1, 0, az), pl.read_raw(2, 0, az))
    st = pl.stats() if hasattr(pl, "stats") else None
    pl.close()
    return out, st


CASES = [
    # nx, ny, nz, n, k: ragged x/y tiles (136 = 2 x 64 + 8, 52 = 3 x 16 + 4), boundary-only and interior chunks
    (136, 52, 96, 1, 1),
    (136, 52, 96, 3, 2),
    (64, 32, 128, 4, 4),
    (200, 72, 64, 2, 3),
    (40, 36, 160, 5, 1),
    # degenerate: the smallest grid (4^2 planes: one tile, 2 x 2 interior blocks), 2kR = 16 > the 12-plane
    # chunk width (extents reach past the neighbour chunk), one chunk spanning the domain
    (4, 4, 16, 2, 1),
    (8, 8, 48, 4, 2),
    (12, 20, 32, 1, 2),
]


@pytest.mark.parametrize("nx,ny,nz,n,k", CASES)
@pytest.mark.parametrize("rate", [16, 8, 12])
def test_fused_first_step_bitwise(nx, ny, nz, n, k, rate):
    steps = 2 * k
    ref, _ = run(nx, ny, nz, n, k, steps, False, rate=rate)
    got, _ = run(nx, ny, nz, n, k, steps, True, rate=rate)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


@pytest.mark.parametrize("mode,store,kw", [
    ("compress", "host", {}),
    ("dwb", "host", {}),
    ("swb", "device", {}),
    ("swb", "device", {"decoded_velocity": True}),
    ("swb", "host", {"resident_velocity": True}),
    ("swb", "host", {"n_lanes": 2}),
    ("swb", "host", {"schedule": "dag"}),
    ("swb", "host", {"schedule": "dag_func", "executor": "split"}),
    # the DAG schedules must order the next H2D into a staging slot after the fused step's read of it (the
    # race checker found this edge missing with the resident velocity, where the encode output no longer
    # overlaps p_{t-1}'s input region)
    ("swb", "host", {"schedule": "dag_func", "resident_velocity": True, "n_lanes": 2}),
    ("dwb", "host", {"schedule": "dag", "resident_velocity": True}),
])
def test_fused_modes_bitwise(mode, store, kw):
    nx, ny, nz, n, k = 136, 52, 128, 4, 2
    ref, _ = run(nx, ny, nz, n, k, 6, False, mode=mode, store=store, **kw)
    got, _ = run(nx, ny, nz, n, k, 6, True, mode=mode, store=store, **kw)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_fused_split_runs_equal_one_run():
    nx, ny, nz, n, k = 72, 40, 96, 3, 2
    ref, _ = run(nx, ny, nz, n, k, 8, False)
    got, _ = run(nx, ny, nz, n, k, 8, True, split=[2, 4, 2])
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


@pytest.mark.parametrize("store", ["host", "device"])
def test_fused_medium_grid_z_split(store):
    # 512^2 planes: 256 tiles < 296 resident CTAs, so the step's z range is split across CTAs (the fused
    # kernel rounds each CTA's z range to whole 4-plane slabs); 4 chunks, k = 4, two sweeps
    nx, ny, nz, n, k = 512, 512, 256, 4, 4
    ref, _ = run(nx, ny, nz, n, k, 8, False, store=store)
    got, _ = run(nx, ny, nz, n, k, 8, True, store=store)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])
