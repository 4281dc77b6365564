"""BASELINE.json configs[2]: temporal-blocking depth sweep k in {1,2,4,8} x rate sweep r in {8,12,16,24}
on 2048^3 fp32 (16 chunks, T = 8 steps), one B200.  For every point: Gcell-updates/s with the state in
HBM (kernel throughput), out-of-core through PCIe (the paper's pipeline), and out-of-core with the
compressed velocity kept resident (OOCS_FLAG_RESIDENT_VELOCITY), with the transfer bytes and the PCIe
roofline -- the crossover from PCIe-bound to kernel-bound the north star asks for.

    python tools/sweep.py [--n 2048] [--ks 1,2,4,8] [--rates 8,12,16,24] [--out profiles/r01_sweep_c3.json]
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

R = 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--nb", type=int, default=16)
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--rates", default="8,12,16,24")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep_c3.json"))
    a = ap.parse_args()
    n, nb, T = a.n, a.nb, a.T
    mb = json.load(open(os.path.join(ROOT, "profiles", "r01_measure_box.json")))
    dt = float(synth.dt_for())
    rows = []
    for r in [int(x) for x in a.rates.split(",")]:
        for k in [int(x) for x in a.ks.split(",")]:
            mk = lambda store, **kw: oocs.Plan(oocs.make_config(nx=n, ny=n, nz=n, dt=dt, n_blocks=nb, tb_depth=k,
                                                                rate_bits=r, mode="swb", store=store, **kw))
            t0 = time.time()
            dev = mk("device")
            bench.load_state(dev, n, n, n, 0)
            dev.run(T)
            sd = dev.run(T)
            row = {"n": n, "k": k, "rate": r, "T": T, "value_gcups": sd.cell_updates / (sd.wall_ms * 1e-3) / 1e9,
                   "device_gb": dev.info.arena_bytes / 1e9}
            host = mk("host")
            bench.copy_state(dev, host)
            dev.close()
            host.run(T)
            sh = host.run(T)
            row["e2e_gcups"] = sh.cell_updates / (sh.wall_ms * 1e-3) / 1e9
            row["h2d_bytes"] = sh.bytes_h2d
            row["d2h_bytes"] = sh.bytes_d2h
            hpc, dpc = sh.bytes_h2d / sh.cell_updates, sh.bytes_d2h / sh.cell_updates
            row["pcie_roofline_gcups"] = 1.0 / max(hpc / mb["h2d_gbs"], dpc / mb["d2h_gbs"],
                                                   (hpc + dpc) / mb["duplex_total_gbs"])
            row["e2e_bound"] = "pcie" if row["pcie_roofline_gcups"] < row["value_gcups"] else "kernel"
            hv = mk("host", resident_velocity=True)
            bench.copy_state(host, hv)
            host.close()
            hv.run(T)
            sv = hv.run(T)
            row["e2e_resident_v_gcups"] = sv.cell_updates / (sv.wall_ms * 1e-3) / 1e9
            hpc = sv.bytes_h2d / sv.cell_updates
            row["pcie_roofline_resident_v_gcups"] = 1.0 / max(hpc / mb["h2d_gbs"], dpc / mb["d2h_gbs"],
                                                              (hpc + dpc) / mb["duplex_total_gbs"])
            row["resident_v_device_gb"] = hv.info.arena_bytes / 1e9
            hv.close()
            row["seconds"] = time.time() - t0
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump({"config": "BASELINE.json configs[2] (2048^3, 16 chunks) k x rate sweep", "rows": rows,
               "pcie": {k: mb[k] for k in ("h2d_gbs", "d2h_gbs", "duplex_total_gbs")}}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
