"""Per-GPU memory of every pipeline mode for the BASELINE.json configs (oocs_plan_estimate: exactly what
oocs_plan_create would allocate, without allocating) -- the paper's GPU-memory experiment
at B200 scale, incl. configs[4]'s single- vs double-working-buffer comparison at 8 GPUs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_11315_b200 as oocs  # noqa: E402

CONFIGS = {
    "c1": dict(nx=64, ny=64, nz=64, n_blocks=4, tb_depth=2, world=1),
    "c2": dict(nx=1024, ny=1024, nz=1024, n_blocks=8, tb_depth=4, world=1),
    "c3_k8": dict(nx=2048, ny=2048, nz=2048, n_blocks=16, tb_depth=8, world=1),
    "c4_1gpu": dict(nx=4096, ny=4096, nz=4096, n_blocks=64, tb_depth=4, world=1),
    "c4_8gpu": dict(nx=4096, ny=4096, nz=4096, n_blocks=64, tb_depth=4, world=8),
    "c5_8gpu": dict(nx=4096, ny=4096, nz=8192, n_blocks=128, tb_depth=4, world=8),
}


def table():
    out = {}
    for name, kw in CONFIGS.items():
        row = {}
        for mode, codec in (("baseline", "identity"), ("compress", "blockquant"), ("swb", "blockquant"),
                            ("dwb", "blockquant")):
            c = oocs.make_config(dt=0.1, codec=codec, rate_bits=16, mode=mode, rank=0, **kw)
            i = oocs.oocs_plan_estimate(c)
            row[mode] = {"device_gb": i.arena_bytes / 1e9, "host_store_gb": i.store_bytes / 1e9,
                         "working_set_gb": i.working_set_bytes / 1e9, "staging_gb": i.staging_bytes / 1e9}
        c = oocs.make_config(dt=0.1, rate_bits=16, mode="swb", store="device", **kw)
        i = oocs.oocs_plan_estimate(c)
        row["device_resident"] = {"device_gb": i.arena_bytes / 1e9}
        row["swb_vs_baseline_reduction"] = 1 - row["swb"]["device_gb"] / row["baseline"]["device_gb"]
        row["swb_vs_dwb_saving_gb"] = row["dwb"]["device_gb"] - row["swb"]["device_gb"]
        out[name] = row
    return out


if __name__ == "__main__":
    t = table()
    print(json.dumps(t, indent=1))
    if "--save" in sys.argv:
        json.dump({"source": "tools/memory_table.py (oocs_plan_estimate, rate 16, per GPU, rank 0)", "table": t},
                  open(os.path.join(ROOT, "profiles", "r01_memory_table.json"), "w"), indent=1)
