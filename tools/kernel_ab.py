"""Same-box A/B of liboocs builds on the HBM-resident pipeline (sustained kernels, no PCIe): for every
library given, a device-store plan (default c3: 2048^3, 16 chunks, k = 4, r = 16) runs --reps oocs_run
calls of T steps with OOCS_FLAG_PROFILE; prints value (Gcell-updates/s) and the per-kernel algorithmic
GB/s.  Libraries alternate (A B A B ...) so clock / power drift hits both.

    OOCS_LIB is set per run: python tools/kernel_ab.py A.so B.so [--wl c3] [--rounds 2] [--reps 3]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
import bench, synth, paper_2204_11315_b200 as oocs
nx, ny, nz, nb, k, T, rate = bench.WORKLOADS[%(wl)r]
k = %(k)s or k
T = %(T)s or T
kw = dict(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=nb, tb_depth=k, rate_bits=%(rate)s or rate,
          mode="swb", store="device", profile=True)
kw.update(%(extra)s)
pl = oocs.Plan(oocs.make_config(**kw))
bench.load_state(pl, nx, ny, nz, 0)
pl.run(T)
best = None
for _ in range(%(reps)s):
    st = pl.run(T)
    if best is None or st.wall_ms < best.wall_ms:
        best = st
out = {"value": best.cell_updates / (best.wall_ms * 1e-3) / 1e9, "wall_ms": best.wall_ms}
for i, name in enumerate(["decode", "step", "encode"]):
    ms = best.kernel_ms[i]
    out[name] = {"ms": ms, "GBps": best.alg_bytes[i] / (ms * 1e-3) / 1e9 if ms else None,
                 "launches": best.kernel_launches[i]}
print(json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--wl", default="c3")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--rate", type=int, default=0)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--extra", default="{}", help="extra make_config kwargs as a Python dict literal")
    a = ap.parse_args()
    code = CHILD % {"root": ROOT, "wl": a.wl, "k": a.k, "T": a.T, "rate": a.rate, "reps": a.reps,
                    "extra": a.extra, "flags": 0}
    for r in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ, OOCS_LIB=os.path.abspath(lib))
            res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if res.returncode:
                print(lib, "FAILED", res.stderr[-2000:])
                continue
            d = json.loads(res.stdout.strip().splitlines()[-1])
            print(json.dumps({"lib": os.path.basename(lib), "round": r, "value": round(d["value"], 2),
                              **{k: (round(d[k]["GBps"] or 0), round(d[k]["ms"], 1)) for k in ("decode", "step", "encode")}}),
                  flush=True)


if __name__ == "__main__":
    main()
