"""PCIe: 1-D pinned copies vs the pitched 2-D copies the uncompressed BASELINE issues (rows of ax*4 B into a
working buffer with a larger pitch), both directions, c2 plane sizes."""
import ctypes
import os
import sys

import torch

cudart = ctypes.CDLL("libcudart.so.12")
ax, ay, planes = 1032, 1032, 160
pitch = (28 + ax + 31) // 32 * 32
rows = ay * planes
host = torch.empty(rows * ax * 4, dtype=torch.uint8).pin_memory()
dev = torch.empty(rows * pitch * 4, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
H2D, D2H = 1, 2


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            fn()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


nbytes = rows * ax * 4
for kind, name in ((H2D, "H2D"), (D2H, "D2H")):
    src, dst = (host, dev) if kind == H2D else (dev, host)
    one = lambda: cudart.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                         ctypes.c_size_t(nbytes), kind, ctypes.c_void_p(st.cuda_stream))
    if kind == H2D:
        two = lambda: cudart.cudaMemcpy2DAsync(ctypes.c_void_p(dev.data_ptr() + 112), ctypes.c_size_t(pitch * 4),
                                               ctypes.c_void_p(host.data_ptr()), ctypes.c_size_t(ax * 4),
                                               ctypes.c_size_t(ax * 4), ctypes.c_size_t(rows), kind,
                                               ctypes.c_void_p(st.cuda_stream))
    else:
        two = lambda: cudart.cudaMemcpy2DAsync(ctypes.c_void_p(host.data_ptr()), ctypes.c_size_t(ax * 4),
                                               ctypes.c_void_p(dev.data_ptr() + 112), ctypes.c_size_t(pitch * 4),
                                               ctypes.c_size_t(ax * 4), ctypes.c_size_t(rows), kind,
                                               ctypes.c_void_p(st.cuda_stream))
    t1, t2 = timeit(one), timeit(two)
    print(f"{name}: 1-D {nbytes / t1 / 1e6:.1f} GB/s, pitched 2-D {nbytes / t2 / 1e6:.1f} GB/s ({nbytes / 1e9:.2f} GB)")
