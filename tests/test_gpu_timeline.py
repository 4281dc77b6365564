"""OOCS_FLAG_TIMELINE on the GPU: one span per work op of the lowered schedule, and the orderings the
schedule promises observed on the device clock -- stream order within a lane, the single-working-buffer
hand-off (decode of chunk g after encode of chunk g-1, Alg. 1), and the cross-sweep
read-after-write on the in-place host store (H2D of chunk i in sweep t+1 after the D2H of chunks i and
i+1 in sweep t)."""
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_11315_b200 as oocs  # noqa: E402

EPS = 2e-3  # ms: event timestamp resolution


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("executor", ["dispatch", "single", "split"])
@pytest.mark.parametrize("sched", ["alg1", "dag"])
@pytest.mark.parametrize("store", ["host", "device"])
def test_timeline_spans_and_orderings(store, sched, executor):
    nx, ny, nz, n, k, T = 64, 64, 96, 4, 2, 6
    vel, p0 = synth.fields(nx, ny, nz)
    az = vel.shape[0]
    c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, rate_bits=16,
                         mode="swb", store=store, schedule=sched, timeline=True, executor=executor)
    pl = oocs.Plan(c)
    for a, arr in enumerate((vel, p0, p0)):
        pl.load(a, arr, 0, az)
    st = pl.run(T)
    spans = pl.timeline()
    ops = [o for o in oocs.oocs_schedule(c, T) if o["kind"] not in ("WAIT", "RECORD")]
    key = lambda x: (x["kind"], x["g"], x["arg"])
    # one span per work op (the dispatcher may issue them in another order than the list)
    assert sorted(map(key, spans)) == sorted(map(key, ops))
    if executor != "dispatch":
        assert list(map(key, spans)) == list(map(key, ops))
    for s in spans:
        assert -EPS <= s["start_ms"] <= s["end_ms"] + EPS and s["end_ms"] <= st.wall_ms + EPS
    # program order within a lane: its ops run one after another, in schedule order
    by = {key(s): s for s in spans}
    for lane in {o["lane"] for o in ops}:
        mine = [by[key(o)] for o in ops if o["lane"] == lane]
        for x, y in zip(mine, mine[1:]):
            assert y["start_ms"] >= x["end_ms"] - EPS
    G = max(s["g"] for s in spans) + 1
    for g in range(1, G):
        # single working buffer: chunk g is decoded only after chunk g-1 was encoded
        assert by[("DECODE", g, 0)]["start_ms"] >= by[("ENCODE", g - 1, 0)]["end_ms"] - EPS
    if store == "host":
        for g in range(n, G):
            i = g % n
            for j in (i, i + 1):
                if j < n:
                    assert by[("H2D", g, 0)]["start_ms"] >= by[("D2H", g - n + (j - i), 0)]["end_ms"] - EPS
    # engine busy times in the stats = union of the spans
    for e, kinds in enumerate((("H2D",), ("D2H",), ("DECODE", "STEP", "ENCODE"))):
        iv = sorted((s["start_ms"], s["end_ms"]) for s in spans if s["kind"] in kinds)
        tot, lo, hi = 0.0, 0.0, -1.0
        for a, b in iv:
            if a > hi:
                tot += max(hi - lo, 0.0)
                lo, hi = a, b
            else:
                hi = max(hi, b)
        tot += max(hi - lo, 0.0)
        assert abs(st.busy_ms[e] - tot) < 1e-3 * max(tot, 1.0)
    # the flag off: no spans
    pl.close()
    c2 = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=n, tb_depth=k, rate_bits=16,
                          mode="swb", store=store, schedule=sched)
    pl = oocs.Plan(c2)
    for a, arr in enumerate((vel, p0, p0)):
        pl.load(a, arr, 0, az)
    pl.run(T)
    assert pl.timeline() == []
    pl.close()
