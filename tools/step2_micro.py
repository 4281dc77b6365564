"""The fused two-step stencil (oocs_step2) against two single steps (oocs_step) on a c3 chunk's working
buffer (2048^2 interior, 168 planes: the first step pair of an interior k = 4 chunk, 152 + 144 planes),
CUDA-event timed: burst (12 launches, median) and sustained (back to back for ~3 s).  Algorithmic bytes:
single step 16 B per computed update; two-step = 16 B per level-t+1 cell (read A, B, v; write C) + 4 B
per level-t+2 cell (write D).

    python tools/step2_micro.py [--n 2048] [--out gpurun_out/step2_micro.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--planes", type=int, default=168)
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "step2_micro.json"))
    a = ap.parse_args()
    nx = ny = a.n
    planes = a.planes
    ax, ay = nx + 2 * R, ny + 2 * R
    pitch = oocs.pitch_for(ax)
    dt = 0.1
    mk = lambda: torch.rand(planes, ay, pitch, device="cuda")
    v = mk() + 1.0
    A, B, C, D = mk(), mk(), mk(), mk()
    st = torch.cuda.current_stream().cuda_stream
    z1 = (R + 4, planes - R - 4)
    z2 = (z1[0] + R, z1[1] - R)
    c1, c2 = (z1[1] - z1[0]) * nx * ny, (z2[1] - z2[0]) * nx * ny

    def two_single():
        oocs.oocs_step(v.data_ptr(), A.data_ptr(), B.data_ptr(), ax, ay, planes, pitch, dt, z1[0], z1[1], st)
        oocs.oocs_step(v.data_ptr(), B.data_ptr(), A.data_ptr(), ax, ay, planes, pitch, dt, z2[0], z2[1], st)

    def fused():
        oocs.oocs_step2(v.data_ptr(), A.data_ptr(), B.data_ptr(), C.data_ptr(), D.data_ptr(), ax, ay, planes, pitch,
                        dt, z1[0], z1[1], z2[0], z2[1], st)

    out = {"n": a.n, "planes": planes, "z1": z1, "z2": z2, "updates": c1 + c2}
    for name, fn, alg in (("two_single_steps", two_single, 16 * (c1 + c2)), ("fused_step2", fused, 16 * c1 + 4 * c2)):
        ts = []
        for i in range(14):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        burst = sorted(ts)[len(ts) // 2]
        n = max(10, int(a.seconds * 1e3 / burst))
        evs = []
        for i in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in evs[n // 2:])
        sus = ms[len(ms) // 2]
        out[name] = {"burst_ms": burst, "sustained_ms": sus, "gcups_burst": (c1 + c2) / burst / 1e6,
                     "gcups_sustained": (c1 + c2) / sus / 1e6, "alg_GBps_burst": alg / burst / 1e6,
                     "alg_GBps_sustained": alg / sus / 1e6, "alg_bytes": alg}
        print(name, json.dumps(out[name]), flush=True)
    out["speedup_sustained"] = out["two_single_steps"]["sustained_ms"] / out["fused_step2"]["sustained_ms"]
    out["speedup_burst"] = out["two_single_steps"]["burst_ms"] / out["fused_step2"]["burst_ms"]
    print("speedup", out["speedup_burst"], out["speedup_sustained"])
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
