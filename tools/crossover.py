"""The PCIe -> kernel-bound crossover the north star asks for ("an end-to-end out-of-core stencil whose
B200 pipeline is bound by kernel throughput rather than PCIe"), on BASELINE.json configs[2]'s grid
(2048^3 fp32, 16 z-chunks of W = 128).

Deeper temporal blocking divides the PCIe bytes per cell-update by k (H2D = 3 (r/8) / k, D2H = 2 (r/8) / k,
SURVEY §8(d)) while the kernels' HBM bytes per update stay ~16 rho + codec/k (rho = 1 + R(k-1)/W): the
paper's lever (P:L85, P:L228-233 fig:newbot -- "GPU kernel time is longer than CPU-GPU data movement time"
after compression).  For every (r, k): the HBM-resident value (kernels only), the out-of-core run (pinned
host store, every byte over PCIe in the timed region) with its per-op timeline (OOCS_FLAG_TIMELINE: busy
fraction of the H2D copies, the D2H copies and the kernels), and the ratio out-of-core / resident.  The
pipeline is kernel-bound where that ratio approaches 1 and the kernel busy fraction approaches 1 while
the H2D busy fraction falls.

    python tools/crossover.py [--rates 8,16] [--ks 4,8,12,16] [--out profiles/r02_crossover_c3.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--nb", type=int, default=16)
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--ks", default="4,8,12,16")
    ap.add_argument("--rates", default="8,16")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_crossover_c3.json"))
    ap.add_argument("--fuse-decode", action="store_true", help="every plan with OOCS_FLAG_FUSE_DECODE")
    a = ap.parse_args()
    n, nb = a.n, a.nb
    dt = float(synth.dt_for())
    link = bench.measure_pcie(0)
    rows = []
    for r in [int(x) for x in a.rates.split(",")]:
        for k in [int(x) for x in a.ks.split(",")]:
            T = a.sweeps * k
            mk = lambda store, **kw: oocs.Plan(oocs.make_config(nx=n, ny=n, nz=n, dt=dt, n_blocks=nb, tb_depth=k,
                                                                rate_bits=r, mode="swb", store=store,
                                                                fuse_decode=a.fuse_decode, **kw))
            t0 = time.time()
            dev = mk("device")
            bench.load_state(dev, n, n, n, 0)
            dev.run(T)
            sd = min((dev.run(T) for _ in range(3)), key=lambda s: s.wall_ms)
            row = {"n": n, "chunks": nb, "k": k, "rate": r, "T": T,
                   "value_device_resident": sd.cell_updates / (sd.wall_ms * 1e-3) / 1e9}
            for label, kw in (("out_of_core", {}), ("out_of_core_resident_v", {"resident_velocity": True})):
                host = mk("host", timeline=True, **kw)
                bench.copy_state(dev, host)
                host.run(T)
                sh = min((host.run(T) for _ in range(3)), key=lambda s: s.wall_ms)
                v = sh.cell_updates / (sh.wall_ms * 1e-3) / 1e9
                hpc, dpc = sh.bytes_h2d / sh.cell_updates, sh.bytes_d2h / sh.cell_updates
                bound = 1.0 / max(hpc / link["h2d_gbs"], dpc / link["d2h_gbs"], (hpc + dpc) / link["duplex_total_gbs"])
                busy = list(sh.busy_ms)
                row[label] = {"value": v, "ratio_to_device_resident": v / row["value_device_resident"],
                              "pcie_bound_gcups": bound, "frac_of_pcie_bound": v / bound,
                              "h2d_bytes_per_update": hpc, "d2h_bytes_per_update": dpc,
                              "busy_frac": {"h2d": busy[0] / sh.wall_ms, "d2h": busy[1] / sh.wall_ms,
                                            "kernels": busy[2] / sh.wall_ms},
                              "bound": "pcie" if bound < row["value_device_resident"] else "kernel",
                              "device_gb": host.info.arena_bytes / 1e9}
                host.close()
            dev.close()
            row["seconds"] = time.time() - t0
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump({"config": f"BASELINE.json configs[2] grid ({n}^3, {nb} chunks, W = {n // nb}), k x rate, "
                         f"{a.sweeps} sweeps per oocs_run, best of 3 runs"
                         + (", decode -> first step fusion (OOCS_FLAG_FUSE_DECODE)" if a.fuse_decode else ""),
               "rows": rows, "pcie": link}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
