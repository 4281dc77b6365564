"""oocs_run_async / oocs_wait: a run issued while the previous one drains (chainable plans: host store,
codec modes, Algorithm 1, one rank) must give bitwise the state of the same steps in blocking oocs_run
calls -- and of one oocs_run of all the steps -- for every mode, lane count and the resident velocity;
the runs' stats come back in issue order and add up; other calls complete the runs in flight first;
plans that cannot chain fall back to run-after-run."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402
from test_gpu_parity import load_fields  # noqa: E402

R = 4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _plan(nx, ny, nz, n, k, **kw):
    kw.setdefault("mode", "swb")
    kw.setdefault("codec", "blockquant")
    return oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k,
                                      rate_bits=16 if kw["codec"] != "identity" else 32, **kw))


CASES = [dict(mode="swb"), dict(mode="swb", n_lanes=2), dict(mode="dwb"), dict(mode="compress", n_lanes=4),
         dict(mode="swb", resident_velocity=True), dict(mode="swb", codec="zfp"), dict(mode="swb", codec="identity")]


@pytest.mark.parametrize("kw", CASES)
@pytest.mark.parametrize("n,k", [(4, 2), (2, 1), (5, 3)])
def test_chained_runs_bitwise(kw, n, k):
    nx, ny, nz = 36, 28, 20 * n
    if kw.get("codec") == "zfp":
        kw = dict(kw, rate_bits=12)
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    steps = [k, 2 * k, k, 3 * k]
    outs = []
    for how in ("one", "sync", "async"):
        pl = _plan(nx, ny, nz, n, k, **{x: y for x, y in kw.items() if x != "rate_bits"})
        load_fields(pl, vel, p0)
        if how == "one":
            pl.run(sum(steps))
        elif how == "sync":
            for s in steps:
                pl.run(s)
        else:
            for s in steps:
                pl.run_async(s)
            st = pl.wait()
            assert len(st) == len(steps)
            assert [x.cell_updates for x in st] == [nx * ny * nz * s for s in steps]
            assert all(x.wall_ms > 0 for x in st)
        outs.append([pl.read_raw(a, 0, az) for a in (1, 2)])
        pl.close()
    for o in outs[1:]:
        for a in range(2):
            assert np.array_equal(o[a], outs[0][a])


def test_async_then_other_calls_complete_the_runs():
    nx, ny, nz, n, k = 32, 24, 64, 4, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    ref = _plan(nx, ny, nz, n, k)
    load_fields(ref, vel, p0)
    ref.run(4 * k)
    want = ref.store(2, 0, az)
    ref.close()
    pl = _plan(nx, ny, nz, n, k)
    load_fields(pl, vel, p0)
    pl.run_async(2 * k)
    pl.run_async(2 * k)
    got = pl.store(2, 0, az)  # completes both runs first
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    st = pl.wait()  # the runs' stats are still reported
    assert len(st) == 2
    pl.run_async(k)
    pl.close()  # destroy completes the run in flight


@pytest.mark.parametrize("kw", [dict(store="device"), dict(schedule="dag"), dict(mode="baseline", codec="identity"),
                                dict(timeline=True), dict(executor="single")])
def test_async_falls_back_where_runs_cannot_chain(kw):
    nx, ny, nz, n, k = 32, 24, 64, 4, 2
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    outs = []
    for asyn in (False, True):
        pl = _plan(nx, ny, nz, n, k, **kw)
        load_fields(pl, vel, p0)
        for _ in range(3):
            if asyn:
                pl.run_async(k)
            else:
                pl.run(k)
        if asyn:
            assert len(pl.wait()) == 3
        outs.append(pl.read_raw(2, 0, az))
        pl.close()
    assert np.array_equal(outs[0], outs[1])


def test_async_data_error_reported_by_wait():
    """A value the encoder must reject (|x| >= 2^126) produced inside a chained run: oocs_wait
    reports OOCS_ERR_DATA (the plan is not poisoned)."""
    nx, ny, nz, n, k = 32, 24, 64, 4, 1
    vel, p0 = synth.fields(nx, ny, nz)
    az = nz + 2 * R
    pp, pc = p0.copy(), p0.copy()
    pp[R + 30, R + 5, R + 5] = -7e37  # p_next = 2 p - p_prev + c L ~ 1.1e38 > 2^126 = 8.5e37
    pc[R + 30, R + 5, R + 5] = 7e37
    pl = _plan(nx, ny, nz, n, k)
    pl.load(0, vel, 0, az)
    pl.load(1, pp, 0, az)
    pl.load(2, pc, 0, az)
    pl.run_async(k)
    pl.run_async(k)
    with pytest.raises(oocs.OocsError) as e:
        pl.wait()
    assert e.value.status == 6
    pl.close()
