"""Pipeline timeline of one out-of-core run (OOCS_FLAG_TIMELINE): the analog of the paper's pipeline
figures (fig:pipe1 P:L100, fig:newbot P:L228), with nsys absent from this image.

Runs the bench workload (c2: 1024^3, 8 chunks, k = 4, T = 16, BlockQuant r = 16, single working buffer)
with the pinned host store, records a CUDA-event span around every op, and reports per engine (H2D,
D2H, kernels) the busy time (union of spans), its fraction of the run, the overlap of the two PCIe
directions, the idle gaps of the H2D engine (where the pipeline stalls), an ASCII Gantt chart, and the
spans themselves.

    python tools/timeline.py [--workload c2] [--codec blockquant] [--resident-velocity] [--out FILE]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402

ENGINES = {"H2D": ("H2D",), "D2H": ("D2H",), "kernel": ("DECODE", "STEP", "ENCODE"), "carry": ("CARRY",)}


def union(iv):
    """Total length of a union of [a, b) intervals, and the merged list."""
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return sum(b - a for a, b in out), out


def intersect_len(x, y):
    i = j = 0
    tot = 0.0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if b > a:
            tot += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return tot


def gantt(merged, wall, width=120):
    rows = {}
    for name, iv in merged.items():
        line = [" "] * width
        for a, b in iv:
            for c in range(int(a / wall * width), min(width, int(b / wall * width) + 1)):
                line[c] = "#"
        rows[name] = "".join(line)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--codec", default="blockquant", choices=["blockquant", "zfp", "trunc16"])
    ap.add_argument("--store", default="host", choices=["host", "device"])
    ap.add_argument("--resident-velocity", action="store_true")
    ap.add_argument("--executor", default="dispatch", choices=["dispatch", "single", "split"],
                    help="host dispatcher (default) or stream replay: one stream per lane (Alg. 1 literal) / "
                         "copy + kernel stream per lane")
    ap.add_argument("--schedule", default="alg1", choices=["alg1", "dag", "dag_func"])
    ap.add_argument("--lanes", type=int, default=0, help="pipeline lanes (0 = 3, Alg. 1's strm[0:3])")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_timeline_c2.json"))
    a = ap.parse_args()
    nx, ny, nz, nb, k, T, rate = bench.WORKLOADS[a.workload]
    if a.codec == "trunc16":
        rate = 16
    cfg = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=nb, tb_depth=k, codec=a.codec,
                           rate_bits=rate, mode="swb", store=a.store, resident_velocity=a.resident_velocity,
                           schedule=a.schedule, timeline=True, n_lanes=a.lanes,
                           executor=a.executor)
    pl = oocs.Plan(cfg)
    bench.load_state(pl, nx, ny, nz, 0)
    pl.run(T)  # warm-up
    st = pl.run(T)
    spans = pl.timeline()
    wall = st.wall_ms
    merged, busy = {}, {}
    for eng, kinds in ENGINES.items():
        busy[eng], merged[eng] = union([(s["start_ms"], s["end_ms"]) for s in spans if s["kind"] in kinds])
    # gaps of the H2D engine longer than 1% of the run: where the PCIe input stream stalls
    gaps = []
    h = merged["H2D"]
    for (a0, b0), (a1, b1) in zip(h, h[1:]):
        if a1 - b0 > 0.01 * wall:
            nxt = next(s for s in spans if s["kind"] == "H2D" and abs(s["start_ms"] - a1) < 1e-9)
            gaps.append({"from_ms": b0, "to_ms": a1, "ms": a1 - b0, "next_h2d": {"sweep": nxt["sweep"],
                                                                                "block": nxt["block"]}})
    head = 0.0 if not h else h[0][0]
    tail = 0.0 if not h else wall - h[-1][1]
    res = {
        "workload": f"{a.workload}: {nx}x{ny}x{nz}, {nb} chunks, k={k}, T={T}, {a.codec} rate {rate}, swb, "
                    f"{a.store} store{', resident velocity' if a.resident_velocity else ''}, schedule {a.schedule}, "
                    f"executor {a.executor}, lanes {a.lanes or 3}",
        "wall_ms": wall,
        "gcell_updates_per_s": st.cell_updates / (wall * 1e-3) / 1e9,
        "bytes_h2d": st.bytes_h2d, "bytes_d2h": st.bytes_d2h,
        "busy_ms": busy, "busy_frac": {e: busy[e] / wall for e in busy},
        "h2d_while_busy_gbs": st.bytes_h2d / (busy["H2D"] * 1e-3) / 1e9 if busy["H2D"] else None,
        "d2h_while_busy_gbs": st.bytes_d2h / (busy["D2H"] * 1e-3) / 1e9 if busy["D2H"] else None,
        "h2d_d2h_overlap_ms": intersect_len(merged["H2D"], merged["D2H"]),
        "kernel_hidden_under_pcie_frac": intersect_len(merged["kernel"], union(
            [tuple(x) for x in merged["H2D"] + merged["D2H"]])[1]) / max(busy["kernel"], 1e-9),
        "h2d_head_ms": head, "h2d_tail_ms": tail, "h2d_gaps": gaps,
        "gantt": gantt(merged, wall),
        "host_enqueue_ms": max(s["host_ms"] for s in spans),
        "spans": [[s["kind"], s["lane"], s["sweep"], s["block"], s["arg"], round(s["start_ms"], 4),
                   round(s["end_ms"], 4), round(s["host_ms"], 4)] for s in spans],
        "spans_columns": ["kind", "lane", "sweep", "block", "step", "start_ms", "end_ms", "host_enqueue_ms"],
    }
    pl.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k not in ("spans", "gantt")}, indent=1))
    for name, line in res["gantt"].items():
        print(f"{name:>7} |{line}|")


if __name__ == "__main__":
    main()
