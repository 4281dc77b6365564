"""Fluid discrete-event simulation of a lowered oocs schedule (tools only, not a test).

Ops run in lane FIFO order after their event waits; kernels share the SMs (one at a
time), H2D / D2H share PCIe (duplex-limited), CARRY is a device copy.  Durations come
from measured rates.  Used to compare schedule variants before spending GPU time."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_11315_b200 as oocs

H2D_BW, D2H_BW, DUPLEX = 55.6e9, 57.2e9, 100.3e9


def simulate(cfg, steps, kernel_ms=(0.21, 0.41, 0.24), d2d_bw=2.5e12, verbose=False):
    ops = oocs.oocs_schedule(cfg, steps)
    blocks = oocs.oocs_plan_table(cfg)
    pb = oocs.oocs_encoded_bytes(cfg, 4) / 4
    nl = 1 + max(o["lane"] for o in ops)
    lanes = [[] for _ in range(nl)]
    for i, o in enumerate(ops):
        lanes[o["lane"]].append(i)
    rec_time = {}
    done = [None] * len(ops)
    pos = [0] * nl
    t = 0.0
    running = {}  # op -> remaining work (bytes or ms)
    sm_busy = None
    def work(o):
        b = blocks[o["block"]]
        if o["kind"] == "H2D":
            return ("h2d", 3 * (b[7] - b[6]) * pb)
        if o["kind"] == "D2H":
            return ("d2h", 2 * (b[1] - b[0]) * pb)
        if o["kind"] == "CARRY":
            return ("d2d", 3 * (b[5] - b[4]) * pb / d2d_bw * 1e3)
        if o["kind"] == "DECODE":
            return ("sm", 3 * kernel_ms[0])
        if o["kind"] == "STEP":
            return ("sm", kernel_ms[1])
        if o["kind"] == "ENCODE":
            return ("sm", 2 * kernel_ms[2])
        return (None, 0)
    busy_h2d = 0.0
    while True:
        progressed = True
        while progressed:
            progressed = False
            for l in range(nl):
                while pos[l] < len(lanes[l]):
                    i = lanes[l][pos[l]]
                    o = ops[i]
                    if i in running:
                        break
                    if o["kind"] == "RECORD":
                        rec_time[(o["ev"], o["ev_g"])] = t; done[i] = t; pos[l] += 1; progressed = True; continue
                    if o["kind"] == "WAIT":
                        key = (o["ev"], o["ev_g"])
                        if key in rec_time and rec_time[key] <= t:
                            done[i] = t; pos[l] += 1; progressed = True; continue
                        # recorded later in issue order? (waits on never-recorded are no-ops)
                        rec_idx = [j for j, p in enumerate(ops) if p["kind"] == "RECORD" and (p["ev"], p["ev_g"]) == key and j < i]
                        if not rec_idx:
                            done[i] = t; pos[l] += 1; progressed = True; continue
                        break
                    res, w = work(o)
                    if res == "sm" and sm_busy is not None:
                        break
                    running[i] = [res, w]
                    if res == "sm":
                        sm_busy = i
                    break
        if not running:
            break
        # rates
        act = {r for r, _ in running.values()}
        h2d_rate = (DUPLEX / 2 if "d2h" in act else H2D_BW)
        d2h_rate = (DUPLEX / 2 if "h2d" in act else D2H_BW)
        n_h2d = sum(1 for r, _ in running.values() if r == "h2d")
        n_d2h = sum(1 for r, _ in running.values() if r == "d2h")
        def rate(r):
            if r == "h2d": return h2d_rate / n_h2d / 1e3  # bytes per ms
            if r == "d2h": return d2h_rate / n_d2h / 1e3
            return 1.0
        dt = min(w / rate(r) for r, w in running.values())
        if "h2d" in act:
            busy_h2d += dt
        t += dt
        fin = []
        for i, (r, w) in list(running.items()):
            running[i][1] = w - dt * rate(r)
            if running[i][1] <= 1e-9:
                fin.append(i)
        for i in fin:
            del running[i]
            done[i] = t
            if sm_busy == i:
                sm_busy = None
            pos[ops[i]["lane"]] += 1
    cells = cfg.nx * cfg.ny * cfg.nz * steps
    return t, cells / (t * 1e-3) / 1e9, busy_h2d / t


if __name__ == "__main__":
    c = oocs.make_config(nx=1024, ny=1024, nz=1024, dt=0.1, n_blocks=8, tb_depth=4, mode="swb")
    t, gc, hb = simulate(c, 16)
    print(f"c2 swb: {t:.1f} ms/step  {gc:.2f} Gcu/s  h2d busy {hb:.2f}")
