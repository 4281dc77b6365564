"""Stencil kernel alone: oocs_step on a c2-sized working buffer (1024^2 interior, 160 planes), launches
back to back, per-launch CUDA-event times; compared with the same launches interleaved with decode and
encode launches as in the pipeline."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4
nx = ny = 1024
planes = 160
ax, ay = nx + 2 * R, ny + 2 * R
pitch = oocs.pitch_for(ax)
dt = 0.1
v = torch.rand(planes, ay, pitch, device="cuda") + 1.0
a = torch.rand(planes, ay, pitch, device="cuda")
b = torch.rand(planes, ay, pitch, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def launch(zlo, zhi):
    oocs.oocs_step(v.data_ptr(), a.data_ptr(), b.data_ptr(), ax, ay, planes, pitch, dt, zlo, zhi, st)


for name, (zlo, zhi), fl in [("152 planes", (R, R + 152), False), ("152 planes, L2 flushed", (R, R + 152), True),
                             ("128 planes", (16, 144), False), ("136 planes", (12, 148), False)]:
    ts = []
    for i in range(12):
        if fl:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch(zlo, zhi)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    alg = (zhi - zlo) * nx * ny * 16
    print(f"{name}: median {ms * 1e3:.1f} us, {alg / ms / 1e6:.0f} GB/s algorithmic, min {min(ts) * 1e3:.1f} us")

# sustained: back-to-back launches for ~4 s; per-launch time early vs late (power cap / clocks)
ts = []
for i in range(9000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch(R, R + 152)
    e1.record()
    ts.append((e0, e1))
    if len(ts) >= 9000 or (i > 100 and sum(1 for _ in ()) > 0):
        break
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in ts]
alg = 152 * nx * ny * 16
for lo, hi in ((0, 50), (1000, 1050), (4000, 4050), (8900, 8950)):
    seg = sorted(ms[lo:hi])
    print(f"sustained launches {lo}-{hi}: median {seg[len(seg) // 2] * 1e3:.1f} us = {alg / seg[len(seg) // 2] / 1e6:.0f} GB/s")
