"""How the PCIe link shares itself between the two directions: a continuous pinned H2D stream (the
out-of-core pipeline's binding direction) against a D2H stream issued at a paced rate (pieces of
--piece MiB released by the host at the target rate; 'full' = back to back).  If the link splits fairly
only when both directions saturate, pacing D2H just above what the pipeline needs (69 GB per 104 GB of
H2D at c3) would let H2D run closer to its solo rate.

    python tools/pcie_pacing.py [--seconds 2] [--piece 32] [--out gpurun_out/pcie_pacing.json]
"""
import argparse
import json
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0)
    ap.add_argument("--piece", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "pcie_pacing.json"))
    a = ap.parse_args()
    n_h2d = 256 << 20
    piece = a.piece << 20
    h = torch.empty(n_h2d, dtype=torch.uint8, pin_memory=True).fill_(1)
    d = torch.empty(n_h2d, dtype=torch.uint8, device="cuda")
    hd = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dd = torch.empty(1 << 30, dtype=torch.uint8, device="cuda").fill_(2)
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    rows = []
    for target in (0, 20, 30, 36, 40, 44, 48, "full"):
        torch.cuda.synchronize()
        stop = threading.Event()
        moved = [0]

        def d2h_pacer():
            t0 = time.perf_counter()
            off = 0
            while not stop.is_set():
                if target != "full":
                    due = t0 + moved[0] / (target * 1e9)
                    now = time.perf_counter()
                    if now < due:
                        time.sleep(min(due - now, 0.002))
                        continue
                with torch.cuda.stream(sd):
                    hd[off:off + piece].copy_(dd[off:off + piece], non_blocking=True)
                moved[0] += piece
                off = (off + piece) % (hd.numel() - piece)
                if target == "full" and moved[0] % (16 * piece) == 0:
                    sd.synchronize()  # keep the queue bounded

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = int(a.seconds * 55e9 / n_h2d)
        th = threading.Thread(target=d2h_pacer) if target != 0 else None
        if th:
            th.start()
            time.sleep(0.05)
        t_start = time.perf_counter()
        with torch.cuda.stream(sh):
            e0.record(sh)
            for _ in range(reps):
                d.copy_(h, non_blocking=True)
            e1.record(sh)
        e1.synchronize()
        t_h2d = e0.elapsed_time(e1) * 1e-3
        wall = time.perf_counter() - t_start
        stop.set()
        if th:
            th.join()
        sd.synchronize()
        row = {"d2h_target_gbs": target, "h2d_gbs": reps * n_h2d / t_h2d / 1e9,
               "d2h_gbs_issued": moved[0] / wall / 1e9 if th else 0.0}
        row["sum_gbs"] = row["h2d_gbs"] + row["d2h_gbs_issued"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump({"piece_mib": a.piece, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
