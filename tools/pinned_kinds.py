"""Pinned host memory kinds against the PCIe link: cudaHostAlloc default vs portable vs write-combined
(1 GiB, best of 8, CUDA events): H2D alone, D2H alone and duplex.  The out-of-core store is pinned with
the default flags; write-combined memory skips the CPU cache snoop on DMA, at the price of uncached CPU
reads.

    python tools/pinned_kinds.py [--out gpurun_out/pinned_kinds.json]
"""
import argparse
import ctypes
import glob
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "pinned_kinds.json"))
    a = ap.parse_args()
    torch.cuda.init()
    libs = sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so.1*")) or sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))
    rt = ctypes.CDLL(libs[0])
    rt.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    rt.cudaFreeHost.argtypes = [ctypes.c_void_p]
    n = 1 << 30
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, flags in (("default", 0), ("portable", 1), ("write_combined", 4)):
        ph, ph2 = ctypes.c_void_p(), ctypes.c_void_p()
        assert rt.cudaHostAlloc(ctypes.byref(ph), n, flags) == 0 and rt.cudaHostAlloc(ctypes.byref(ph2), n, flags) == 0
        ctypes.memset(ph, 1, n)
        ctypes.memset(ph2, 2, n)

        def bw(fn, moved):
            best = 0.0
            for _ in range(8):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s1)
                fn()
                s1.wait_stream(s2)
                e1.record(s1)
                torch.cuda.synchronize()
                best = max(best, moved / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            return best

        h2d = lambda st, src=ph: rt.cudaMemcpyAsync(d.data_ptr(), src, n, 1, ctypes.c_void_p(st.cuda_stream))
        d2h = lambda st, dst=ph2: rt.cudaMemcpyAsync(dst, d2.data_ptr(), n, 2, ctypes.c_void_p(st.cuda_stream))

        def duplex():
            s2.wait_stream(s1)
            h2d(s1)
            d2h(s2)

        out[name] = {"h2d_gbs": bw(lambda: h2d(s1), n), "d2h_gbs": bw(lambda: d2h(s1), n),
                     "duplex_total_gbs": bw(duplex, 2 * n)}
        print(name, json.dumps(out[name]), flush=True)
        rt.cudaFreeHost(ph)
        rt.cudaFreeHost(ph2)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
