"""The fused two-step stencil (oocs_step2, NEXT-2 temporal register blocking) against two single steps
(oocs_step) -- bitwise: it performs the same IEEE operations in the same order -- and against two oracle
steps within the per-step 1e-6 bar.  Interior-chunk ranges (step 2's range R planes inside step 1's) and
boundary ranges (both steps to the Dirichlet planes), grids spanning several 64 x 16 tiles with ragged
x / y tails, and a z range long enough to be split across CTAs; C / D must be untouched outside the
interior cells of their ranges."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from test_gpu_parity import _rel_err, from_ws, stream, to_ws  # noqa: E402

R = 4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def _fields(nx, ny, nz, seed):
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(seed)
    pp = (p0 * np.float32(0.95) + rng.normal(scale=1e-2, size=p0.shape).astype(np.float32)).astype(np.float32)
    pp[:R], pp[-R:], pp[:, :R], pp[:, -R:], pp[:, :, :R], pp[:, :, -R:] = 0, 0, 0, 0, 0, 0  # Dirichlet halo = B's
    return vel, np.ascontiguousarray(pp), p0


@pytest.mark.parametrize("shape,kind", [((100, 36, 40), "interior"), ((100, 36, 40), "boundary"),
                                        ((200, 72, 120), "interior"), ((64, 16, 24), "boundary"),
                                        ((136, 20, 200), "interior")])
def test_step2_bitwise_equals_two_steps(shape, kind):
    nx, ny, nz = shape
    vel, A, B = _fields(nx, ny, nz, nz)
    az, ay, ax = B.shape
    pitch = oocs.pitch_for(ax)
    dt = synth.dt_for()
    if kind == "interior":
        z1 = (R + 8, az - R - 8)
        z2 = (z1[0] + R, z1[1] - R)
    else:
        z1 = z2 = (R, az - R)
    tv, ta, tb = to_ws(vel), to_ws(A), to_ws(B)
    tc = torch.full_like(ta, float("nan"))
    td = torch.full_like(ta, float("nan"))
    oocs.oocs_step2(tv.data_ptr(), ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), td.data_ptr(), ax, ay, az, pitch, dt,
                    z1[0], z1[1], z2[0], z2[1], stream())
    # reference: two single steps in place
    ra, rb = to_ws(A), to_ws(B)
    oocs.oocs_step(tv.data_ptr(), ra.data_ptr(), rb.data_ptr(), ax, ay, az, pitch, dt, z1[0], z1[1], stream())
    oocs.oocs_step(tv.data_ptr(), rb.data_ptr(), ra.data_ptr(), ax, ay, az, pitch, dt, z2[0], z2[1], stream())
    torch.cuda.synchronize()
    C, D, RA, RB = (from_ws(t, ax) for t in (tc, td, ra, rb))
    i1 = (slice(z1[0], z1[1]), slice(R, ay - R), slice(R, ax - R))
    i2 = (slice(z2[0], z2[1]), slice(R, ay - R), slice(R, ax - R))
    assert np.array_equal(C[i1].view(np.uint32), RA[i1].view(np.uint32))
    assert np.array_equal(D[i2].view(np.uint32), RB[i2].view(np.uint32))
    # untouched outside the interior cells of the ranges
    mc = np.ones(C.shape, bool)
    mc[i1] = False
    md = np.ones(D.shape, bool)
    md[i2] = False
    assert np.all(np.isnan(C[mc])) and np.all(np.isnan(D[md]))
    # and within the bar of two oracle steps
    oa, ob = A.copy(), B.copy()
    oracle.step(vel, oa, ob, dt, z1[0], z1[1])
    oracle.step(vel, ob, oa, dt, z2[0], z2[1])
    assert _rel_err(D[i2], ob[i2].astype(np.float64)) <= 2e-6


def test_step2_rejects_bad_ranges():
    nx, ny, nz = 64, 16, 40
    vel, A, B = _fields(nx, ny, nz, 1)
    az, ay, ax = B.shape
    t = [to_ws(x) for x in (vel, A, B, B, B)]
    p = [x.data_ptr() for x in t]
    pitch = oocs.pitch_for(ax)
    for z1, z2 in [((R, 30), (R + 5, 26)),   # step 2 more than R planes inside step 1
                   ((R + 4, 30), (R, 26)),   # step 2 starts below step 1
                   ((R - 1, 30), (R + 3, 26))]:
        with pytest.raises(oocs.OocsError):
            oocs.oocs_step2(p[0], p[1], p[2], p[3], p[4], ax, ay, az, pitch, 0.1, z1[0], z1[1], z2[0], z2[1], stream())
    with pytest.raises(oocs.OocsError):  # aliasing D with B
        oocs.oocs_step2(p[0], p[1], p[2], p[3], p[2], ax, ay, az, pitch, 0.1, R + 4, 30, R + 8, 26, stream())
