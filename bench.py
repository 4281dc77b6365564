#!/usr/bin/env python
"""Benchmark of the out-of-core compressed stencil hot path (arXiv 2204.11315) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl oocs|reference]

One "step" = one oocs_run of the whole hot path over the BASELINE.json configs[1]
workload (c2: 1024^3 fp32 per GPU, 8 z-chunks, 16 time steps = 4 sweeps of
temporal depth k=4, BlockQuant rate 16 bits/value, single working buffer):
every chunk is decompressed, advanced k steps on the shrinking trapezoid and
recompressed, every sweep.

* value: Gcell-updates/s with the compressed state resident in HBM when the timed
  region starts (store="device"; no PCIe) -- the kernels' throughput;
* e2e:   the same metric through the C ABI with the compressed state in pinned HOST
  memory (store="host", the paper's out-of-core pipeline): H2D of every chunk body,
  GPU decode / steps / encode, D2H of the owned planes, on 3 streams (Alg. 1).
N > 1 (torchrun): weak scaling, rank r owns a 1024^3 z-slab of a 1024x1024x(1024N)
grid; inter-slab halos are exchanged with NCCL after each sweep.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

R = 4
METRIC = "out-of-core Gcell-updates/s incl. transfers; roofline %; peak GPU memory (GB)"
UNIT = "Gcell-updates/s"
WORKLOADS = {
    # name: (nx, ny, nz per rank, chunks per rank, k, T, rate)
    "c2": (1024, 1024, 1024, 8, 4, 16, 16),
    "c1": (64, 64, 64, 4, 2, 4, 16),
    # configs[3] per GPU: 4096^2 x 512 planes, 8 chunks of W = 64 per rank, k = 4, T = 32; at --gpus 8
    # this is c4 itself (4096^3, 64 chunks); on one GPU it is one rank's weak-scaling share
    "c4slab": (4096, 4096, 512, 8, 4, 32, 16),
}


def env_int(k, d):
    return int(os.environ.get(k, d))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)  # >= 5 timed repetitions
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="oocs", choices=["oocs", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fuse-encode", action="store_true", help="fuse each chunk's last step with its encode "
                    "(device store, BlockQuant; OOCS_FLAG_FUSE_ENCODE)")
    ap.add_argument("--no-compare", action="store_true", help="skip the uncompressed / memory comparison")
    ap.add_argument("--codec", default="blockquant", choices=["blockquant", "zfp", "trunc16"],
                    help="fixed-rate codec of the compressed state (ZFP = NEXT-1)")
    ap.add_argument("--schedule", default="alg1", choices=["alg1", "dag", "dag_func"],
                    help="stream/event schedule of the host-store pipeline (e2e)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with several ranks sharing one GPU")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def smi_mem_used_mib(device):
    """Device memory in use (MiB) per nvidia-smi: the cross-check of a plan's arena bytes (SURVEY 8(d):
    arena bytes + NVML memory.used delta).  None when nvidia-smi is unavailable."""
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(device), "--query-gpu=memory.used",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20).stdout
        return int(out.strip().splitlines()[0])
    except Exception:
        return None


def measure_pcie(device, nbytes=1 << 30, reps=8):
    """Pinned H2D / D2H / duplex bandwidth of THIS box's link (best of `reps`, CUDA events), measured
    before the timed regions, so the e2e PCIe roofline is this box's and not another's (the method of
    tools/measure_box.py, smaller)."""
    import torch

    dev = torch.device("cuda", device)
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def bw(fn, moved):
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            with torch.cuda.stream(s):
                e0.record(s)
                fn()
                e1.record(s)
            torch.cuda.synchronize(dev)
            best = max(best, moved / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        return best

    def duplex():
        s2.wait_stream(s)
        d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        s.wait_stream(s2)

    out = {"h2d_gbs": bw(lambda: d.copy_(h, non_blocking=True), nbytes),
           "d2h_gbs": bw(lambda: h2.copy_(d, non_blocking=True), nbytes),
           "duplex_total_gbs": bw(duplex, 2 * nbytes), "source": f"live, this box ({nbytes >> 20} MiB pinned copies)"}
    del h, h2, d, d2
    return out


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def load_state(plan, nx, ny, nz_global, device):
    """Generate the synthetic fields slab by slab on the GPU (synth.fields_torch), compress them into
    the plan's store through oocs_load (outside any timed region)."""
    import synth

    info = plan.info
    a_lo, a_hi = info.store_lo + R, info.store_hi + R
    slab = 64
    for z0 in range(a_lo, a_hi, slab):
        z1 = min(a_hi, z0 + slab)
        v, p = synth.fields_torch(nx, ny, nz_global, z0, z1, device=f"cuda:{device}")
        v, p = v.cpu().numpy(), p.cpu().numpy()
        plan.load(0, v, z0, z1)
        plan.load(1, p, z0, z1)
        plan.load(2, p, z0, z1)


def copy_state(src, dst):
    a_lo, a_hi = src.info.store_lo + R, src.info.store_hi + R
    for a in range(3):
        dst.write_raw(a, src.read_raw(a, a_lo, a_hi), a_lo, a_hi)


def timed_runs(plan, T, steps, warmup, barrier, clocks=None):
    for _ in range(warmup):
        plan.run(T)
    barrier()
    per = []
    wall0 = time.perf_counter()
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        for _ in range(steps):
            per.append(plan.run(T))
    wall = time.perf_counter() - wall0
    barrier()
    return per, wall


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def step_summary(stats_list):
    """Per timed step device ms (median and best of the repetitions, with all of them)."""
    ms = sorted(s.wall_ms for s in stats_list)
    return {"median": float(np.median(ms)), "best": ms[0], "all": [round(s.wall_ms, 3) for s in stats_list]}


def agg(stats_list):
    out = {"ms": sum(s.wall_ms for s in stats_list), "kernel_ms": [0.0] * 3, "launches": [0] * 3,
           "alg": [0] * 3, "h2d": 0, "d2h": 0, "cells": 0, "computed": 0, "exch": 0}
    for s in stats_list:
        for i in range(3):
            out["kernel_ms"][i] += s.kernel_ms[i]
            out["launches"][i] += s.kernel_launches[i]
            out["alg"][i] += s.alg_bytes[i]
        out["h2d"] += s.bytes_h2d
        out["d2h"] += s.bytes_d2h
        out["cells"] += s.cell_updates
        out["computed"] += s.cell_updates_computed
        out["exch"] += s.bytes_exchange
    return out


# ----------------------------------------------------------------------------- CPU oracle timing
ORACLE_CODEC = {"blockquant": (1, lambda r: r - 1), "zfp": (2, lambda r: r), "trunc16": (3, lambda r: 0)}
CODEC_NAME = {"blockquant": "BlockQuant", "zfp": "ZFP", "trunc16": "Truncate-16 (bf16)"}


def cpu_oracle_sample(nx, ny, k, rate, device=None, codec="blockquant"):
    """Bounded sample of the workload through the CPU oracle: a nx*ny*256 slab (two of c2's
    128-plane chunks, interior-size trapezoids), one sweep of k steps, the same codec and rate."""
    import oracle
    import synth

    nz = 256
    if device is not None:
        v, p = synth.fields_torch(nx, ny, nz, device=device)
        v, p = v.cpu().numpy(), p.cpu().numpy()
    else:
        v, p = synth.fields(nx, ny, nz)
    cid, qf = ORACLE_CODEC[codec]
    q = qf(rate)
    S = [oracle.encode_planes(a, cid, q) for a in (v, p, p)]
    ax, ay = nx + 2 * R, ny + 2 * R
    dt = synth.dt_for()

    def one():
        Sp, Sc = S[1].copy(), S[2].copy()
        t0 = time.perf_counter()
        oracle.pipeline(ax, ay, nz, 2, k, dt, k, cid, q, S[0], Sp, Sc)
        return time.perf_counter() - t0

    cells = nx * ny * nz * k
    sample = f"CPU oracle pipeline on a {nx}x{ny}x{nz} slab (2 chunks of 128 planes), 1 sweep of k={k} steps, {CODEC_NAME[codec]} rate {rate}"
    return one, cells, sample


def threads_used():
    """Host cores the oracle runs on: every core of the affinity mask.  torchrun exports
    OMP_NUM_THREADS=1 for its ranks; the oracle legs run on rank 0 alone, so they are widened back to
    the whole host (oracle.set_threads), and this is the count they actually use."""
    return len(os.sched_getaffinity(0))


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    nx, ny, nzr, nbr, k, T, rate = WORKLOADS[args.workload]
    if args.codec == "trunc16":
        rate = 16  # bfloat16
    import torch

    nz = nzr * world
    nblocks = nbr * world
    workload = (f"{args.workload}: {nx}x{ny}x{nz} fp32 interior (+4-cell halo), {nblocks} z-chunks, {T} steps, "
                f"temporal depth k={k}, {CODEC_NAME[args.codec]} rate {rate} bits/value, "
                f"single working buffer")
    config = {"workload": workload, "nx": nx, "ny": ny, "nz": nz, "n_blocks": nblocks, "tb_depth": k,
              "time_steps_per_step": T, "rate_bits": rate, "codec": args.codec, "mode": "swb",
              "fused_last_step_encode": args.codec == "blockquant" and args.fuse_encode,
              "parallelism": f"z-slabs x{world}",
              "l2": f"inputs larger than L2 (compressed state {3 * nx * ny * nzr * rate / 8 / 1e9:.1f} GB/GPU >> 126 MB), "
                    "no flush needed"}

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle

        oracle.set_threads(threads_used())
        one, cells, sample = cpu_oracle_sample(nx, ny, k, rate,
                                               device="cuda" if torch.cuda.is_available() else None,
                                               codec=args.codec)
        for _ in range(args.warmup):
            one()
        secs = sum(one() for _ in range(args.steps))
        v = cells * args.steps / secs / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 stencil / f32 codec",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads_used(), "kind": "oracle",
                                 "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    dist = None
    gloo = args.dist_backend == "gloo"
    if world > 1:
        import torch.distributed as dist

        if gloo:
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if gloo else "cuda"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if dist is None:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        return float(t.item())

    import paper_2204_11315_b200 as oocs
    from paper_2204_11315_b200 import dist as odist

    dt = float(__import__("synth").dt_for())

    def mk(store, mode="swb", codec=None, profile=False, resident_velocity=False, decoded_velocity=False):
        codec = codec or args.codec
        c = oocs.make_config(nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nblocks, tb_depth=k, codec=codec,
                             rate_bits=rate, mode=mode, store=store, device=local, rank=rank, world=world,
                             profile=profile, resident_velocity=resident_velocity, schedule=args.schedule,
                             fusion=args.fuse_encode, decoded_velocity=decoded_velocity)
        pl = oocs.Plan(c)
        if world > 1:
            pl.set_exchange((odist.gloo_exchange_fn if gloo else odist.nccl_exchange_fn)(rank, world))
        return pl

    peak_gbs, peak_src = measured_peaks()
    out = {}

    # ---- value: compressed state resident in HBM -------------------------------------------
    dev = mk("device", profile=True)
    load_state(dev, nx, ny, nz, local)
    clocks = ClockSampler(local)
    per, wall = timed_runs(dev, T, args.steps, args.warmup, barrier, clocks)
    a = agg(per)
    dev_ms = allmax(a["ms"])
    cells_all = allsum(a["cells"])
    value = cells_all / (dev_ms * 1e-3) / 1e9
    mem_dev = dev.info.arena_bytes
    # roofline of the dominant kernel (largest summed launch time)
    names = ["decode", "step", "encode"]
    kdom = int(np.argmax(a["kernel_ms"]))
    launches = max(1, a["launches"][kdom])
    achieved = a["alg"][kdom] / (a["kernel_ms"][kdom] * 1e-3) / 1e9
    ncu = ncu_traffic()
    traffic = None
    if ncu and names[kdom] in ncu:
        # DRAM bytes / algorithmic bytes of the profiled launch (ncu --set full), scaled to this run's
        # average launch
        traffic = ncu[names[kdom]]["traffic_over_alg"] * a["alg"][kdom] / launches
    roofline = {"bound": "hbm", "kernel": names[kdom], "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                "traffic_source": "profiles/ncu_summary.json (dram__bytes_read+write of one ncu --set full launch)",
                "alg_bytes_per_launch": a["alg"][kdom] / launches,
                "avg_launch_ms": a["kernel_ms"][kdom] / launches,
                "share_of_step": a["kernel_ms"][kdom] / a["ms"] if a["ms"] else None,
                "per_kernel": {names[i]: {"ms": a["kernel_ms"][i], "launches": a["launches"][i],
                                          "GBps": (a["alg"][i] / (a["kernel_ms"][i] * 1e-3) / 1e9)
                                          if a["kernel_ms"][i] else None} for i in range(3)}}
    gpu_launches = int(sum(a["launches"]))
    clk = clocks.summary()
    # variant: the read-only velocity kept decoded in HBM (OOCS_FLAG_DECODED_VELOCITY): each chunk decodes
    # two arrays instead of three; bitwise the same results (tests/test_gpu_parity.py)
    cfg_dv = dict(store="device", profile=True, decoded_velocity=True)
    need = oocs.oocs_plan_estimate(oocs.make_config(
        nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nblocks, tb_depth=k, codec=args.codec, rate_bits=rate, mode="swb",
        store="device", device=local, rank=rank, world=world, decoded_velocity=True)).arena_bytes
    fits = need < torch.cuda.mem_get_info(local)[0] - (2 << 30)
    if world > 1:  # every rank takes the same branch
        fits = allsum(0.0 if fits else 1.0) == 0.0
    if fits:
        dv = mk(**cfg_dv)
        copy_state(dev, dv)
        per_dv, _ = timed_runs(dv, T, args.steps, args.warmup, barrier)
        adv = agg(per_dv)
        dv_ms = allmax(adv["ms"])
        value_dv = {"value": allsum(adv["cells"]) / (dv_ms * 1e-3) / 1e9, "unit": UNIT,
                    "peak_gpu_mem_gb": dv.info.arena_bytes / 1e9,
                    "decode_GBps": adv["alg"][0] / (adv["kernel_ms"][0] * 1e-3) / 1e9 if adv["kernel_ms"][0] else None}
        dv.close()
    else:
        value_dv = {"value": None, "skipped": f"needs {need / 1e9:.1f} GB beside the value plan"}

    # ---- e2e: compressed state in pinned host memory, PCIe in the timed region -------------
    try:
        pcie_live = measure_pcie(local)
    except Exception as exc:  # the committed measurement stands in (reported as such)
        print(f"bench: live PCIe probe failed ({exc}); using profiles/r01_measure_box.json", file=sys.stderr)
        pcie_live = None
    torch.cuda.synchronize(local)
    smi0 = smi_mem_used_mib(local)
    host = mk("host")
    smi1 = smi_mem_used_mib(local)
    smi_delta_gb = (smi1 - smi0) * 2**20 / 1e9 if smi0 is not None and smi1 is not None else None
    copy_state(dev, host)
    dev.close()
    per_h, wall_h = timed_runs(host, T, args.steps, args.warmup, barrier)
    ah = agg(per_h)
    host_ms = allmax(ah["ms"])
    e2e_value = allsum(ah["cells"]) / (host_ms * 1e-3) / 1e9
    mem_swb = host.info.arena_bytes
    # variant: compressed velocity kept resident in HBM (OOCS_FLAG_RESIDENT_VELOCITY, SPEC S:L508 flag)
    hv = mk("host", resident_velocity=True)
    copy_state(host, hv)
    per_v, _ = timed_runs(hv, T, args.steps, 1, barrier)
    av = agg(per_v)
    hv_ms = allmax(av["ms"])
    e2e_resident_v = {"value": allsum(av["cells"]) / (hv_ms * 1e-3) / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": av["h2d"] // args.steps, "d2h_bytes_per_step": av["d2h"] // args.steps,
                      "peak_gpu_mem_gb": hv.info.arena_bytes / 1e9}
    hv.close()
    pcie_bound = pcie_bound_5050 = None
    meas = os.path.join(ROOT, "profiles", "r01_measure_box.json")
    mb = pcie_live
    if mb is None and os.path.exists(meas):
        mb = dict(json.load(open(meas)), source="profiles/r01_measure_box.json (another box)")
    if mb is not None:
        # PCIe roofline of the pipeline: per useful cell-update it must move h2d_pc bytes in and
        # d2h_pc bytes out; time >= max(in/B_h2d, out/B_d2h, (in+out)/B_duplex) (measured links)
        h2d_pc = ah["h2d"] / ah["cells"]
        d2h_pc = ah["d2h"] / ah["cells"]
        t_pc = max(h2d_pc / mb["h2d_gbs"], d2h_pc / mb["d2h_gbs"], (h2d_pc + d2h_pc) / mb["duplex_total_gbs"])
        pcie_bound = 1.0 / t_pc
        # if concurrent H2D+D2H split the measured duplex rate evenly, the best schedule overlaps the
        # smaller direction completely and streams the rest alone:
        lo_, hi_ = min(h2d_pc, d2h_pc), max(h2d_pc, d2h_pc)
        bhi = mb["h2d_gbs"] if h2d_pc >= d2h_pc else mb["d2h_gbs"]
        pcie_bound_5050 = 1.0 / (lo_ / (mb["duplex_total_gbs"] / 2) + (hi_ - lo_) / bhi)
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": ah["h2d"] // args.steps,
           "d2h_bytes_per_step": ah["d2h"] // args.steps, "ms_per_step": host_ms / args.steps,
           "store": "pinned host (PCIe Gen5)", "schedule": args.schedule, "pcie_roofline_gcups": pcie_bound,
           "pcie_frac": (e2e_value / world / pcie_bound) if pcie_bound else None,
           "pcie_roofline_5050_gcups": pcie_bound_5050 if pcie_bound else None,
           "pcie_frac_5050": (e2e_value / world / pcie_bound_5050) if pcie_bound else None,
           "h2d_gbs_achieved": ah["h2d"] / (ah["ms"] * 1e-3) / 1e9,
           "pcie_link": {k: mb[k] for k in ("h2d_gbs", "d2h_gbs", "duplex_total_gbs", "source")} if mb else None,
           "resident_velocity_variant": e2e_resident_v}

    # ---- paper comparisons: uncompressed pipeline (fig:3ver(a)) and peak memory per mode --------
    compare = {}
    if not args.no_compare:
        mem = {"compress_swb": mem_swb, "device_resident": mem_dev}
        for mode in ("compress", "dwb"):
            p = mk("host", mode=mode)
            mem["compress" if mode == "compress" else "compress_dwb"] = p.info.arena_bytes
            p.close()
        base = mk("host", mode="baseline", codec="identity")
        mem["baseline"] = base.info.arena_bytes
        load_state(base, nx, ny, nz, local)
        host.close()
        per_b, _ = timed_runs(base, T, 1, 1, barrier)
        ab = agg(per_b)
        base_ms = allmax(ab["ms"])
        base_value = allsum(ab["cells"]) / (base_ms * 1e-3) / 1e9
        base.close()
        compare = {"uncompressed_baseline_e2e": base_value, "speedup_compressed_vs_uncompressed": e2e_value / base_value,
                   "paper_speedup_v100": 1.1,
                   "peak_gpu_mem_gb": {m: v / 1e9 for m, v in mem.items()},
                   "mem_reduction_swb_vs_baseline": 1 - mem["compress_swb"] / mem["baseline"],
                   "paper_mem_reduction_v100": 0.33}
    else:
        host.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.set_threads(threads_used())
        one, cells, sample = cpu_oracle_sample(nx, ny, k, rate, device=f"cuda:{local}", codec=args.codec)
        # repeat the bounded sample until >= 10 s of CPU work (each repeat restarts from the same state)
        secs, reps = 0.0, 0
        while secs < 10.0 and reps < 16:
            secs += one()
            reps += 1
        cpu = {"value": reps * cells / secs / 1e9, "unit": UNIT, "cores": threads_used(), "kind": "oracle",
               "sample": f"{sample}, x{reps}", "seconds": secs}
        # the same oracle on one core, on a quarter-width slab (all cores and 1 core)
        one1, cells1, sample1 = cpu_oracle_sample(nx // 4, ny // 4, k, rate, device=f"cuda:{local}",
                                                  codec=args.codec)
        oracle.set_threads(1)
        try:
            s1 = one1()
        finally:
            oracle.set_threads(threads_used())
        cpu["one_core"] = {"value": cells1 / s1 / 1e9, "unit": UNIT, "cores": 1, "sample": sample1,
                           "seconds": s1}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "clocks": clk,
                "peak_gpu_mem_gb": mem_swb / 1e9, "peak_gpu_mem_smi_delta_gb": smi_delta_gb,
                "value_store": "device-resident compressed state (HBM)",
                "value_peak_gpu_mem_gb": mem_dev / 1e9, "value_decoded_velocity_variant": value_dv,
                "step_ms_rank0": {"value": step_summary(per), "e2e": step_summary(per_h)},
                "host_wall_s": wall, "compare": compare,
                "cell_updates_computed_per_useful": a["computed"] / a["cells"]}
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
