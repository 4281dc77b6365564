#!/usr/bin/env python
"""Benchmark of the out-of-core compressed stencil hot path (arXiv 2204.11315) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--workload c3|c2|c4slab|beyond_hbm] [--impl oocs|reference]

One "step" = one oocs_run of the whole hot path over the workload: every z-chunk's compressed body
crosses PCIe from the pinned host store (H2D), is decompressed, advanced k steps on the shrinking
trapezoid in the single working buffer, recompressed, and its owned planes go back (D2H), overlapped on
three streams (Algorithm 1).  Default workload: BASELINE.json configs[2]'s headline point
c3 = 2048^3 fp32, 16 z-chunks, k = 4, BlockQuant rate 16 bits/value, T = 8 steps per oocs_run.

* value: out-of-core Gcell-updates/s INCLUDING the transfers (BASELINE.json's metric): useful
  nx*ny*nz*T per step / device time of the K steps (CUDA events on the plan's streams, first H2D of the
  first step to last D2H of the last; the steps are issued back to back with oocs_run_async, each one
  starting while the previous drains), max over ranks.  The compressed state lives in pinned host memory when the timed region
  starts; every byte of it crosses PCIe inside the timed region, every step.
* e2e: the same through the C ABI timed by the host clock around the K oocs_run calls (barrier +
  synchronize on both sides): host dispatch, the H2D of every step's inputs and the D2H of its
  results included.
* value_device_resident: the compressed state resident in HBM (NEXT-2): kernels only.
* roofline: the stencil kernel (event-timed launches inside the timed region) against the measured
  HBM copy peak; roofline_pcie: value against the PCIe link measured live on the box.
* error_vs_incore: max abs error and PSNR of the final p_curr against an uncompressed in-core run of
  the same number of steps on the GPU (oocs_step over the whole grid; bitwise equal to the oracle's
  in-core run, tests/test_gpu_parity.py).
N > 1 (torchrun, or --gpus N which re-launches itself under torchrun): weak scaling, rank r owns a
z-slab of the workload's size; the inter-slab halos go GPU to GPU through peer memory.
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
    # configs[2]'s headline point (k = 4, r = 16, T = 8): the default workload
    "c3": (2048, 2048, 2048, 16, 4, 8, 16),
    "c2": (1024, 1024, 1024, 8, 4, 16, 16),
    "c1": (64, 64, 64, 4, 2, 4, 16),
    # raw state 3 x 4104^2 x 1032 x 4 B = 208 GB > the B200's 192 GB of HBM: out-of-core for real
    # (compressed host store 104 GB at rate 16)
    "beyond_hbm": (4096, 4096, 1024, 8, 4, 8, 16),
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
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-error", action="store_true", help="skip the in-core error run")
    ap.add_argument("--no-device-resident", action="store_true", help="skip the HBM-resident variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true", help="skip the uncompressed / memory comparison")
    ap.add_argument("--codec", default="blockquant", choices=["blockquant", "zfp", "trunc16"],
                    help="fixed-rate codec of the compressed state (ZFP = NEXT-1)")
    # 2 lanes: the same throughput as Alg. 1's three streams on every workload (profiles/r02_lanes.json:
    # c3 33.01 vs 33.01) with one half-size staging buffer less, -20% device memory
    ap.add_argument("--lanes", type=int, default=2, help="pipeline lanes of the compressed modes (Alg. 1's strm[0:3] "
                    "= 3; each lane owns one half-size staging buffer)")
    ap.add_argument("--sync-steps", action="store_true", help="blocking oocs_run per step instead of "
                    "oocs_run_async (no overlap of one step's drain with the next step's fill)")
    ap.add_argument("--schedule", default="alg1", choices=["alg1", "dag", "dag_func"],
                    help="stream/event schedule of the host-store pipeline (e2e)")
    ap.add_argument("--fuse-decode", action="store_true", help="OOCS_FLAG_FUSE_DECODE: the first step of each "
                    "chunk reads p_{t-1} from its compressed records (decode -> first step fusion, NEXT-2)")
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
    """Generate the synthetic fields slab by slab on the GPU (synth.fields_torch) and compress them into
    the plan's store straight from device memory (oocs_load_device), outside any timed region."""
    import synth

    info = plan.info
    a_lo, a_hi = info.store_lo + R, info.store_hi + R
    slab = 64
    for z0 in range(a_lo, a_hi, slab):
        z1 = min(a_hi, z0 + slab)
        v, p = synth.fields_torch(nx, ny, nz_global, z0, z1, device=f"cuda:{device}")
        plan.load_device(0, v.contiguous(), z0, z1)
        plan.load_device(1, p.contiguous(), z0, z1)
        plan.load_device(2, p.contiguous(), z0, z1)
        del v, p


def copy_state(src, dst, slab=128):
    """Raw compressed state from one plan's store to another's, `slab` planes at a time (bounded host
    memory: eight ranks of one node copy at once)."""
    a_lo, a_hi = src.info.store_lo + R, src.info.store_hi + R
    for a in range(3):
        for z0 in range(a_lo, a_hi, slab):
            z1 = min(a_hi, z0 + slab)
            dst.write_raw(a, src.read_raw(a, z0, z1), z0, z1)


def step_summary(stats_list):
    """Per timed step device ms (median and best of the repetitions, with all of them)."""
    ms = sorted(s.wall_ms for s in stats_list)
    return {"median": float(np.median(ms)), "best": ms[0], "all": [round(s.wall_ms, 3) for s in stats_list]}


def agg(stats_list):
    out = {"ms": sum(s.wall_ms for s in stats_list), "kernel_ms": [0.0] * 3, "launches": [0] * 3,
           "alg": [0] * 3, "h2d": 0, "d2h": 0, "cells": 0, "computed": 0, "exch": 0, "copy_launches": 0}
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
        out["copy_launches"] += s.copy_launches
    return out


# ----------------------------------------------------------------------------- CPU oracle timing
ORACLE_CODEC = {"blockquant": (1, lambda r: r - 1), "zfp": (2, lambda r: r), "trunc16": (3, lambda r: 0)}
CODEC_NAME = {"blockquant": "BlockQuant", "zfp": "ZFP", "trunc16": "Truncate-16 (bf16)"}


def cpu_oracle_sample(nx, ny, k, rate, device=None, codec="blockquant", nz=128):
    """Bounded sample of the workload through the CPU oracle: one nx*ny*nz z-chunk (the workload's
    chunk width; one chunk with its own Dirichlet ends), one sweep of k steps, the same codec and rate."""
    import oracle
    import synth

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
        oracle.pipeline(ax, ay, nz, 1, k, dt, k, cid, q, S[0], Sp, Sc)
        return time.perf_counter() - t0

    cells = nx * ny * nz * k
    sample = (f"CPU oracle pipeline on one {nx}x{ny}x{nz} z-chunk (decode, k={k} steps, encode), "
              f"{CODEC_NAME[codec]} rate {rate}")
    return one, cells, sample


def threads_used():
    """Host cores the oracle runs on: every core of the affinity mask.  torchrun exports
    OMP_NUM_THREADS=1 for its ranks; the oracle legs run on rank 0 alone, so they are widened back to
    the whole host (oracle.set_threads), and this is the count they actually use."""
    return len(os.sched_getaffinity(0))


# ----------------------------------------------------------------------------- main
def relaunch_under_torchrun(n):
    """--gpus N without torchrun's environment: re-launch this command as N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def host_mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def incore_error(plan, nx, ny, nz, steps, device, dt):
    """error_vs_incore: the same initial fields advanced `steps` steps in core, uncompressed, with the
    library's own stencil kernel over the whole grid (oocs_step; bitwise the oracle's in-core run), then
    max |p_ooc - p_incore| and PSNR = 20 log10((max_ref - min_ref) / RMSE) over the interior of the
    final p_curr (Q22).  Needs 3 uncompressed arrays in HBM."""
    import torch

    import paper_2204_11315_b200 as oocs
    import synth

    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    pitch = oocs.pitch_for(ax)
    dev = torch.device("cuda", device)
    ws = [torch.zeros((az, ay, pitch), dtype=torch.float32, device=dev) for _ in range(3)]
    slab = 64
    for z0 in range(0, az, slab):
        z1 = min(az, z0 + slab)
        v, p = synth.fields_torch(nx, ny, nz, z0, z1, device=f"cuda:{device}")
        ws[0][z0:z1, :, oocs.XOFF:oocs.XOFF + ax] = v
        ws[1][z0:z1, :, oocs.XOFF:oocs.XOFF + ax] = p
        ws[2][z0:z1, :, oocs.XOFF:oocs.XOFF + ax] = p
        del v, p
    st = torch.cuda.current_stream(dev).cuda_stream
    a, b = 1, 2  # a = level t-1, b = level t; oocs_step writes level t+1 into a
    for _ in range(steps):
        oocs.oocs_step(ws[0].data_ptr(), ws[a].data_ptr(), ws[b].data_ptr(), ax, ay, az, pitch, dt, R, az - R, st)
        a, b = b, a
    torch.cuda.synchronize(dev)
    ref = ws[b]
    del ws[0]
    mx_abs, sse, rmax, rmin, n = 0.0, 0.0, -float("inf"), float("inf"), 0
    buf = torch.empty((slab, ay, ax), dtype=torch.float32, device=dev)
    for z0 in range(R, az - R, slab):
        z1 = min(az - R, z0 + slab)
        got = buf[:z1 - z0]
        plan.store_device(2, got, z0, z1)
        r = ref[z0:z1, R:ay - R, oocs.XOFF + R:oocs.XOFF + ax - R].double()
        d = got[:, R:ay - R, R:ax - R].double() - r
        mx_abs = max(mx_abs, float(d.abs().max()))
        sse += float((d * d).sum())
        rmax, rmin = max(rmax, float(r.max())), min(rmin, float(r.min()))
        n += d.numel()
    del ref, buf, ws
    torch.cuda.empty_cache()
    rmse = (sse / n) ** 0.5
    import math
    psnr = 20 * math.log10((rmax - rmin) / rmse) if rmse > 0 else float("inf")
    return {"max_abs": mx_abs, "psnr_db": psnr, "rmse": rmse, "ref_range": [rmin, rmax], "steps": steps,
            "array": "p_curr (level T), interior cells",
            "reference": "uncompressed in-core run on the GPU (oocs_step over the whole grid)"}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    nx, ny, nzr, nbr, k, T, rate = WORKLOADS[args.workload]
    if args.codec == "trunc16":
        rate = 16  # bfloat16
    import torch

    def describe(nzr, nbr):
        nz, nblocks = nzr * world, nbr * world
        workload = (f"{args.workload}: {nx}x{ny}x{nz} fp32 interior (+4-cell halo), {nblocks} z-chunks, {T} steps "
                    f"per step, temporal depth k={k}, {CODEC_NAME[args.codec]} rate {rate} bits/value, single "
                    f"working buffer, {args.lanes} pipeline lanes, compressed state in pinned host memory "
                    f"(out-of-core, PCIe in the timed region)")
        raw_gb = 3 * (nx + 2 * R) * (ny + 2 * R) * (nzr + 2 * R) * 4 / 1e9
        config = {"workload": workload, "nx": nx, "ny": ny, "nz": nz, "n_blocks": nblocks, "tb_depth": k,
                  "time_steps_per_step": T, "rate_bits": rate, "codec": args.codec, "mode": "swb",
                  "store": "pinned host", "raw_state_gb_per_gpu": raw_gb, "lanes": args.lanes,
                  "parallelism": f"z-slabs x{world}",
                  "l2": f"inputs larger than L2 (compressed state {3 * nx * ny * nzr * rate / 8 / 1e9:.1f} GB/GPU "
                        ">> 126 MB, streamed over PCIe every step), no flush needed"}
        return nz, nblocks, config

    nz, nblocks, config = describe(nzr, nbr)

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle

        oracle.set_threads(threads_used())
        one, cells, sample = cpu_oracle_sample(nx, ny, k, rate,
                                               device="cuda" if torch.cuda.is_available() else None,
                                               codec=args.codec, nz=nzr // nbr)
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
    else:
        torch.cuda.set_device(local)
    red_dev = "cpu" if gloo else "cuda"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allred(x, op):
        if dist is None:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    allmax = lambda x: allred(x, dist.ReduceOp.MAX) if dist else x
    allsum = lambda x: allred(x, dist.ReduceOp.SUM) if dist else x

    import paper_2204_11315_b200 as oocs
    from paper_2204_11315_b200 import dist as odist

    dt = float(__import__("synth").dt_for())

    def mk(store, mode="swb", codec=None, profile=False, resident_velocity=False, decoded_velocity=False,
           wl=None, fuse=None):
        codec = codec or args.codec
        wnx, wny, wnz, wnb = (nx, ny, nz, nblocks) if wl is None else wl
        c = oocs.make_config(nx=wnx, ny=wny, nz=wnz, dt=dt, n_blocks=wnb, tb_depth=k, codec=codec,
                             rate_bits=rate if codec != "identity" else 32, mode=mode, store=store, device=local,
                             rank=rank if wl is None else 0, world=world if wl is None else 1,
                             profile=profile, resident_velocity=resident_velocity, schedule=args.schedule,
                             decoded_velocity=decoded_velocity, n_lanes=0 if mode == "baseline" else args.lanes,
                             fuse_decode=(args.fuse_decode if fuse is None else fuse) and mode != "baseline"
                             and codec == "blockquant")
        pl = oocs.Plan(c)
        if world > 1 and wl is None:
            odist.connect(pl, gloo=gloo)
        return pl

    peak_gbs, peak_src = measured_peaks()

    # ---- the out-of-core plan: compressed state in pinned host memory ------------------------------
    est = oocs.oocs_plan_estimate(oocs.make_config(
        nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nblocks, tb_depth=k, codec=args.codec, rate_bits=rate, mode="swb",
        store="host", device=local, rank=rank, world=world, n_lanes=args.lanes))
    avail = host_mem_available()
    local_ranks = env_int("LOCAL_WORLD_SIZE", world)
    if avail is not None and est.store_bytes * local_ranks > 0.8 * avail and nbr > 1:
        # weak scaling on a node whose host RAM cannot pin every rank's full slab: fewer chunks of the same
        # width per rank (the per-chunk work, k, r and T unchanged), said so in the config
        fit = int(nbr * 0.8 * avail / (est.store_bytes * local_ranks))
        if fit >= 1:
            full = (nzr, nbr)
            nzr, nbr = nzr // nbr * fit, fit
            nz, nblocks, config = describe(nzr, nbr)
            config["host_ram_limited"] = {"per_rank_full": {"nz": full[0], "chunks": full[1]},
                                          "per_rank_run": {"nz": nzr, "chunks": nbr},
                                          "host_mem_available_gb": avail / 1e9, "local_ranks": local_ranks}
            print(f"bench: host RAM fits {fit} of {full[1]} chunks per rank; running {nzr} planes per rank",
                  file=sys.stderr)
            est = oocs.oocs_plan_estimate(oocs.make_config(
                nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nblocks, tb_depth=k, codec=args.codec, rate_bits=rate,
                mode="swb", store="host", device=local, rank=rank, world=world, n_lanes=args.lanes))
    if avail is not None and est.store_bytes * local_ranks > 0.9 * avail:
        print(f"bench: the pinned host stores need {est.store_bytes * local_ranks / 1e9:.1f} GB, the host has "
              f"{avail / 1e9:.1f} GB available", file=sys.stderr)
        sys.exit(3)
    try:
        pcie_live = measure_pcie(local)
    except Exception as exc:  # the committed measurement stands in (reported as such)
        print(f"bench: live PCIe probe failed ({exc}); using profiles/r01_measure_box.json", file=sys.stderr)
        pcie_live = None
    torch.cuda.synchronize(local)
    smi0 = smi_mem_used_mib(local)
    host = mk("host", profile=True)
    smi1 = smi_mem_used_mib(local)
    smi_delta_gb = (smi1 - smi0) * 2**20 / 1e9 if smi0 is not None and smi1 is not None else None
    t_load = time.perf_counter()
    load_state(host, nx, ny, nz, local)
    t_load = time.perf_counter() - t_load
    # the K steps are issued back to back (oocs_run_async: each run starts while the previous one drains,
    # overlapping the pipeline's fill and drain at every step boundary; bitwise the same state) and
    # completed by oocs_wait; each run's device time counts from the previous run's end, so the K add up
    # to the device time from the first step's start to the last step's end
    for _ in range(args.warmup):
        host.run_async(T)
    host.wait()
    clocks = ClockSampler(local)
    barrier()
    t0 = time.perf_counter()
    with clocks:
        if args.sync_steps:
            per = [host.run(T) for _ in range(args.steps)]
        else:
            for _ in range(args.steps):
                host.run_async(T)
            per = host.wait()
        barrier()
        # the host clock stops here: stopping the nvidia-smi sampler (it finishes its current query
        # first, up to ~1 s) is not part of the K steps
        host_wall = time.perf_counter() - t0
    a = agg(per)
    dev_ms = allmax(a["ms"])
    wall_ms = allmax(host_wall * 1e3)
    cells_all = allsum(a["cells"])
    value = cells_all / (dev_ms * 1e-3) / 1e9
    e2e_value = cells_all / (wall_ms * 1e-3) / 1e9
    mem_swb = host.info.arena_bytes
    clk = clocks.summary()
    # roofline of the stencil kernel inside the timed region (event-timed launches, OOCS_FLAG_PROFILE)
    names = ["decode", "step", "encode"]
    kd = 1
    launches = max(1, a["launches"][kd])
    achieved = a["alg"][kd] / (a["kernel_ms"][kd] * 1e-3) / 1e9
    ncu = ncu_traffic()
    traffic = None
    if ncu and names[kd] in ncu:
        traffic = ncu[names[kd]]["traffic_over_alg"] * a["alg"][kd] / launches
    roofline = {"bound": "hbm", "kernel": "stencil_step_tma_kernel", "achieved": achieved, "peak": peak_gbs,
                "unit": "GB/s", "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                "traffic_source": "profiles/ncu_summary.json (dram__bytes_read+write of one ncu --set full launch, "
                                  "scaled to this run's average launch)",
                "alg_bytes_per_launch": a["alg"][kd] / launches, "alg_bytes_per_unit": 16,
                "unit_of_work": "computed cell-update (read p, p_prev, v; write p_next)",
                "avg_launch_ms": a["kernel_ms"][kd] / launches,
                "kernel_busy_share_of_step": sum(a["kernel_ms"]) / a["ms"] if a["ms"] else None,
                "per_kernel": {names[i]: {"ms": a["kernel_ms"][i], "launches": a["launches"][i],
                                          "GBps": (a["alg"][i] / (a["kernel_ms"][i] * 1e-3) / 1e9)
                                          if a["kernel_ms"][i] else None} for i in range(3)}}
    gpu_launches = int(sum(a["launches"]) + a["copy_launches"])  # codec / stencil kernels + SM carry copies
    # PCIe roofline of the pipeline: per useful cell-update it must move h2d_pc bytes in and d2h_pc out;
    # time >= max(in/B_h2d, out/B_d2h, (in+out)/B_duplex) on the link measured live on this box
    mb = pcie_live
    meas = os.path.join(ROOT, "profiles", "r01_measure_box.json")
    if mb is None and os.path.exists(meas):
        mb = dict(json.load(open(meas)), source="profiles/r01_measure_box.json (another box)")
    roofline_pcie = None
    if mb is not None:
        h2d_pc, d2h_pc = a["h2d"] / a["cells"], a["d2h"] / a["cells"]
        t_pc = max(h2d_pc / mb["h2d_gbs"], d2h_pc / mb["d2h_gbs"], (h2d_pc + d2h_pc) / mb["duplex_total_gbs"])
        lo_, hi_ = min(h2d_pc, d2h_pc), max(h2d_pc, d2h_pc)
        bhi = mb["h2d_gbs"] if h2d_pc >= d2h_pc else mb["d2h_gbs"]
        bound_5050 = 1.0 / (lo_ / (mb["duplex_total_gbs"] / 2) + (hi_ - lo_) / bhi)
        moved = (a["h2d"] + a["d2h"]) / (a["ms"] * 1e-3) / 1e9
        roofline_pcie = {"bound": "pcie", "achieved": moved, "peak": mb["duplex_total_gbs"], "unit": "GB/s",
                         "frac": moved / mb["duplex_total_gbs"],
                         "bound_gcups": 1.0 / t_pc, "frac_of_bound": value / world / (1.0 / t_pc),
                         "bound_5050_gcups": bound_5050, "frac_of_bound_5050": value / world / bound_5050,
                         "h2d_gbs_achieved": a["h2d"] / (a["ms"] * 1e-3) / 1e9,
                         "d2h_gbs_achieved": a["d2h"] / (a["ms"] * 1e-3) / 1e9,
                         "bytes_per_cell_update": {"h2d": h2d_pc, "d2h": d2h_pc},
                         "link": {kk: mb[kk] for kk in ("h2d_gbs", "d2h_gbs", "duplex_total_gbs", "source")}}
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": a["h2d"] // args.steps,
           "d2h_bytes_per_step": a["d2h"] // args.steps, "ms_per_step": wall_ms / args.steps,
           "timed": "host clock around the K oocs_run calls through the C ABI (barrier + synchronize both sides)",
           "store": "pinned host (PCIe Gen5)", "schedule": args.schedule,
           "load_s": t_load}

    # ---- error vs an uncompressed in-core run of the same steps (N = 1) -----------------------------
    error = None
    if not args.no_error and world == 1:
        need = 3 * (nz + 2 * R) * (ny + 2 * R) * oocs.pitch_for(nx + 2 * R) * 4
        if need < torch.cuda.mem_get_info(local)[0] - (4 << 30):
            error = incore_error(host, nx, ny, nz, (args.warmup + args.steps) * T, local, dt)
        else:
            error = {"skipped": f"the uncompressed in-core reference needs {need / 1e9:.0f} GB of HBM "
                                f"(raw state exceeds the GPU: that is the out-of-core case)"}

    # ---- variant: compressed state resident in HBM (NEXT-2), kernels only ----------------------------
    value_dev = None
    if not args.no_device_resident:
        torch.cuda.empty_cache()  # the synthetic generator's cached blocks
        need = oocs.oocs_plan_estimate(oocs.make_config(
            nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nblocks, tb_depth=k, codec=args.codec, rate_bits=rate,
            mode="swb", store="device", device=local, rank=rank, world=world)).arena_bytes
        fits = need < torch.cuda.mem_get_info(local)[0] - (2 << 30)
        if world > 1:
            fits = allsum(0.0 if fits else 1.0) == 0.0
        if fits:
            dvp = mk("device", profile=True)
            copy_state(host, dvp)
            for _ in range(min(args.warmup, 3)):
                dvp.run(T)
            barrier()
            per_d = [dvp.run(T) for _ in range(args.steps)]
            barrier()
            ad = agg(per_d)
            d_ms = allmax(ad["ms"])
            value_dev = {"value": allsum(ad["cells"]) / (d_ms * 1e-3) / 1e9, "unit": UNIT,
                         "ms_per_step": d_ms / args.steps, "peak_gpu_mem_gb": dvp.info.arena_bytes / 1e9,
                         "stencil_GBps": ad["alg"][1] / (ad["kernel_ms"][1] * 1e-3) / 1e9,
                         "stencil_frac": ad["alg"][1] / (ad["kernel_ms"][1] * 1e-3) / 1e9 / peak_gbs,
                         "decode_GBps": ad["alg"][0] / (ad["kernel_ms"][0] * 1e-3) / 1e9,
                         "encode_GBps": ad["alg"][2] / (ad["kernel_ms"][2] * 1e-3) / 1e9,
                         "kernel_share_of_step": sum(ad["kernel_ms"]) / ad["ms"]}
            dvp.close()
            # the same with the decode -> first step fusion (OOCS_FLAG_FUSE_DECODE, NEXT-2): bitwise the same
            # state, p_{t-1} read from its records inside the first step
            if args.codec == "blockquant" and rate <= 16 and rate % 2 == 0 and not args.fuse_decode:
                dvf = mk("device", profile=True, fuse=True)
                copy_state(host, dvf)
                for _ in range(min(args.warmup, 3)):
                    dvf.run(T)
                barrier()
                per_f = [dvf.run(T) for _ in range(args.steps)]
                barrier()
                af = agg(per_f)
                f_ms = allmax(af["ms"])
                vf = allsum(af["cells"]) / (f_ms * 1e-3) / 1e9
                value_dev["fused_first_step"] = {
                    "value": vf, "unit": UNIT, "ms_per_step": f_ms / args.steps, "vs_unfused": vf / value_dev["value"],
                    "kernel_ms": dict(zip(["decode", "step", "encode"], af["kernel_ms"])),
                    "unfused_kernel_ms": dict(zip(["decode", "step", "encode"], ad["kernel_ms"])),
                    "flag": "OOCS_FLAG_FUSE_DECODE (opt-in; --fuse-decode runs every plan of the bench with it)"}
                dvf.close()
        else:
            value_dev = {"value": None, "skipped": f"needs {need / 1e9:.1f} GB of HBM"}
    # ---- variant: the read-only velocity kept compressed in HBM (OOCS_FLAG_RESIDENT_VELOCITY):
    #      out-of-core for the two pressures only (2/3 of the H2D bytes); world 1 (host RAM for two stores)
    value_resv = None
    if world == 1 and not args.no_device_resident and host_mem_available() and \
            est.store_bytes < 0.4 * host_mem_available():
        rv = mk("host", resident_velocity=True, profile=True)
        copy_state(host, rv)
        host.close()
        rv.run(T)
        for _ in range(args.steps):
            rv.run_async(T)
        per_v = rv.wait()
        av = agg(per_v)
        value_resv = {"value": av["cells"] / (av["ms"] * 1e-3) / 1e9, "unit": UNIT,
                      "ms_per_step": av["ms"] / args.steps, "peak_gpu_mem_gb": rv.info.arena_bytes / 1e9,
                      "h2d_bytes_per_step": av["h2d"] / args.steps,
                      "note": "out-of-core pressures, compressed velocity resident in HBM (not the paper's accounting)"}
        rv.close()
    else:
        host.close()

    # ---- the paper's two experiments on configs[1] (c2): uncompressed vs compressed, memory ----------
    compare = {}
    if not args.no_compare and world == 1:
        cnx, cny, cnz, cnb, ck, cT, _ = WORKLOADS["c2"]
        wl = (cnx, cny, cnz, cnb)
        runs = {}
        for name, mode, codec in (("compressed_swb", "swb", None), ("uncompressed_baseline", "baseline", "identity")):
            p = mk("host", mode=mode, codec=codec, wl=wl)
            load_state(p, cnx, cny, cnz, local)
            p.run(cT)
            st = [p.run(cT) for _ in range(3)]
            runs[name] = {"value": sum(x.cell_updates for x in st) / (sum(x.wall_ms for x in st) * 1e-3) / 1e9,
                          "peak_gpu_mem_gb": p.info.arena_bytes / 1e9}
            p.close()
        mem = {}
        for wname, (wx, wy, wz, wb) in (("c2", wl), (args.workload, (nx, ny, nz, nblocks))):
            for mode in ("baseline", "compress", "swb", "dwb"):
                base_mode = mode == "baseline"
                cc = oocs.make_config(nx=wx, ny=wy, nz=wz, dt=dt, n_blocks=wb, tb_depth=k,
                                      codec="identity" if base_mode else args.codec, rate_bits=32 if base_mode else rate,
                                      mode=mode, store="host", device=local)
                mem.setdefault(wname, {})[mode] = oocs.oocs_plan_estimate(cc).arena_bytes / 1e9
            cc = oocs.make_config(nx=wx, ny=wy, nz=wz, dt=dt, n_blocks=wb, tb_depth=k, codec=args.codec,
                                  rate_bits=rate, mode="swb", store="host", device=local, n_lanes=2)
            mem[wname]["swb_2_lanes"] = oocs.oocs_plan_estimate(cc).arena_bytes / 1e9
        compare = {"workload": f"c2 (configs[1]): {cnx}x{cny}x{cnz}, {cnb} chunks, k={ck}, T={cT}",
                   "compressed_e2e": runs["compressed_swb"]["value"],
                   "uncompressed_baseline_e2e": runs["uncompressed_baseline"]["value"],
                   "speedup_compressed_vs_uncompressed": runs["compressed_swb"]["value"] / runs["uncompressed_baseline"]["value"],
                   "paper_speedup_v100": 1.1, "peak_gpu_mem_gb_by_mode": mem,
                   "mem_reduction_swb_vs_baseline": {w: 1 - m["swb"] / m["baseline"] for w, m in mem.items()},
                   "mem_reduction_swb_2_lanes_vs_baseline": {w: 1 - m["swb_2_lanes"] / m["baseline"]
                                                             for w, m in mem.items()},
                   "paper_mem_reduction_v100": 0.33}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.set_threads(threads_used())
        one, cells, sample = cpu_oracle_sample(nx, ny, k, rate, device=f"cuda:{local}", codec=args.codec,
                                               nz=nzr // nbr)
        secs, reps = 0.0, 0
        while secs < 10.0 and reps < 16:
            secs += one()
            reps += 1
        cpu = {"value": reps * cells / secs / 1e9, "unit": UNIT, "cores": threads_used(), "kind": "oracle",
               "sample": f"{sample}, x{reps}", "seconds": secs}
        one1, cells1, sample1 = cpu_oracle_sample(nx // 4, ny // 4, k, rate, device=f"cuda:{local}",
                                                  codec=args.codec, nz=nzr // nbr)
        oracle.set_threads(1)
        try:
            s1 = one1()
        finally:
            oracle.set_threads(threads_used())
        cpu["one_core"] = {"value": cells1 / s1 / 1e9, "unit": UNIT, "cores": 1, "sample": sample1, "seconds": s1}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config, "roofline": roofline, "roofline_pcie": roofline_pcie, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk,
                "peak_gpu_mem_gb": mem_swb / 1e9, "peak_gpu_mem_smi_delta_gb": smi_delta_gb,
                "value_store": "pinned host memory (out-of-core; every step's H2D and D2H inside the timed region)",
                "value_device_resident": value_dev, "value_resident_velocity": value_resv, "error_vs_incore": error,
                "step_ms_rank0": step_summary(per), "compare": compare,
                "cell_updates_computed_per_useful": a["computed"] / a["cells"],
                "bytes_exchange_per_step": a["exch"] // args.steps}
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
