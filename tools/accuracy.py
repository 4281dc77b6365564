"""NEXT-3: long-run accuracy of on-the-fly compression (the paper defers it to prior work, P:L214
">4,000 time steps").  The synthetic model on n^3 is advanced to `--steps` (default 4096) with the state
in HBM, BlockQuant at rates 8/12/16/24 and temporal depth k, against the identity codec (which is
bitwise the plain in-core fp32 run, tests/test_gpu_parity.py).  Reports max |error|, RMSE and PSNR of the
current pressure at checkpoints.

    python tools/accuracy.py [--n 512] [--steps 4096] [--out profiles/r01_accuracy.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402
import synth  # noqa: E402

R = 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--nb", type=int, default=8)
    ap.add_argument("--steps", type=int, default=4096)
    ap.add_argument("--ks", default="1,4")
    ap.add_argument("--rates", default="8,12,16,24")
    ap.add_argument("--codec", default="blockquant", choices=["blockquant", "zfp", "trunc16"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_accuracy.json"))
    a = ap.parse_args()
    n, nb = a.n, a.nb
    dt = float(synth.dt_for())
    az = n + 2 * R
    checkpoints = [c for c in (16, 64, 256, 1024, 2048, 4096, 8192) if c <= a.steps]
    rows = []
    for k in [int(x) for x in a.ks.split(",")]:
        mk = lambda codec, r: oocs.Plan(oocs.make_config(nx=n, ny=n, nz=n, dt=dt, n_blocks=nb, tb_depth=k,
                                                         codec=codec, rate_bits=r, mode="swb", store="device"))
        ref = mk("identity", 32)
        bench.load_state(ref, n, n, n, 0)
        lossy = {}
        for r in [int(x) for x in a.rates.split(",")]:
            lossy[r] = mk(a.codec, r)
            bench.load_state(lossy[r], n, n, n, 0)
        done = 0
        for c in checkpoints:
            t0 = time.time()
            ref.run(c - done)
            pr = ref.store(2, 0, az).astype(np.float64)[R:-R, R:-R, R:-R]
            span = pr.max() - pr.min()
            for r, pl in lossy.items():
                pl.run(c - done)
                pg = pl.store(2, 0, az).astype(np.float64)[R:-R, R:-R, R:-R]
                err = pg - pr
                rmse = float(np.sqrt(np.mean(err ** 2)))
                row = {"n": n, "k": k, "codec": a.codec, "rate": r, "steps": c, "max_abs_err": float(np.abs(err).max()),
                       "rmse": rmse, "psnr_db": float(20 * np.log10(span / rmse)) if rmse > 0 else None,
                       "ref_range": float(span), "ref_max_abs": float(np.abs(pr).max())}
                rows.append(row)
                print(json.dumps(row), flush=True)
            done = c
            print(f"# checkpoint {c} ({time.time() - t0:.1f}s)", flush=True)
        ref.close()
        for pl in lossy.values():
            pl.close()
    json.dump({"model": "synth layered velocity + 8 Gaussian pulses + background waves, Dirichlet 0 halo",
               "reference": "identity codec (bitwise the in-core fp32 run)", "rows": rows},
              open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
