"""Measure the GPU box: pinned PCIe H2D/D2H/duplex bandwidth, host RAM, cores."""
import json, os, subprocess, time
import torch

def bw(fn, nbytes, reps=10):
    best = 0.0
    s = torch.cuda.Stream()
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s); fn(s); e1.record(s)
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best

out = {}
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
out["h2d_gbs"] = bw(lambda s: d.copy_(h, non_blocking=True), n)
out["d2h_gbs"] = bw(lambda s: h2.copy_(d, non_blocking=True), n)
s2 = torch.cuda.Stream()
def duplex(s):
    # H2D on s and D2H on s2, both released by the same point of s
    s2.wait_stream(s)
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s.wait_stream(s2)
out["duplex_total_gbs"] = bw(duplex, 2 * n)
out["d2d_copy_gbs"] = bw(lambda s: d2.copy_(d), 2 * n)
for size in (1 << 20, 16 << 20, 256 << 20):
    out[f"h2d_gbs_{size>>20}MiB"] = bw(lambda s: d[:size].copy_(h[:size], non_blocking=True), size)
mi = open("/proc/meminfo").read().split("\n")[:3]
out["meminfo"] = mi
out["cores_affinity"] = len(os.sched_getaffinity(0))
out["cpu_count"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.split("\n")[:25]
except Exception as e:
    out["lscpu"] = str(e)
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm,memory.total", "--format=csv"], capture_output=True, text=True).stdout
# host memcpy bandwidth (single thread numpy)
import numpy as np
a = np.ones(1 << 28, dtype=np.float32); b = np.empty_like(a)
t = time.perf_counter(); np.copyto(b, a); dt = time.perf_counter() - t
out["host_memcpy_1thread_gbs"] = 2 * a.nbytes / dt / 1e9
# multi-threaded host copy bandwidth (the 8-GPU bound needs host DRAM bandwidth; numpy's
# copy releases the GIL, every thread copies its own 512 MiB pair of buffers), and the same while the GPU
# streams duplex over PCIe (the DMA engines read and write the same DRAM)
import threading
def mt_copy(nthreads, secs=1.0):
    bufs = [(np.ones(1 << 27, dtype=np.float32), np.empty(1 << 27, dtype=np.float32)) for _ in range(nthreads)]
    done = [0] * nthreads
    def worker(i):
        a_, b_ = bufs[i]
        t_end = time.perf_counter() + secs
        while time.perf_counter() < t_end:
            np.copyto(b_, a_)
            done[i] += 1
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(nthreads)]
    t0 = time.perf_counter()
    for t_ in ths: t_.start()
    for t_ in ths: t_.join()
    el = time.perf_counter() - t0
    return sum(done) * 2 * bufs[0][0].nbytes / el / 1e9
out["host_memcpy_gbs_by_threads"] = {n_: mt_copy(n_) for n_ in (1, 2, 4, 8, out["cores_affinity"])}
try:
    out["numa_nodes"] = sorted(os.listdir("/sys/devices/system/node"))
except Exception as e:
    out["numa_nodes"] = str(e)
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/measure_box.json", "w"), indent=1)
