"""profiles/ncu_summary.json (bench.py's roofline.traffic source) from the three ncu --set full captures of
tools/gpu_final.sh: DRAM bytes vs algorithmic bytes of the same launch, per kernel.

usage: python tools/make_ncu_summary.py STEP.ncu-rep DECODE.ncu-rep ENCODE.ncu-rep STEP_PLANES
   or: python tools/make_ncu_summary.py --chunk CHUNK.ncu-rep   (one capture of an interior c2 chunk's six
       launches, tools/gpu_round2.sh: decode, steps 1-4 (152/144/136/128 planes), encode)
Algorithmic bytes: stencil 16 B per cell-update (STEP_PLANES x 1024^2); codec (r/8 + 4) B per value,
values = 4 * grid.z planes x 1032^2 (grid z = array x slab)."""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from ncu_summary import summarise  # noqa: E402

RATE = 16
AX = 1032  # c2 (1024 + 2R); --c3: 2056
NX = 1024


def entry(rep, alg, unit, idx=0):
    e = summarise(rep)[idx]
    e["alg_bytes_per_launch"] = alg
    e["alg_unit"] = unit
    e["dram_bytes_per_launch"] = e["dram_bytes"]
    e["traffic_over_alg"] = e["dram_bytes"] / alg
    e["alg_gbs"] = alg / (e["duration_us"] * 1e-6) / 1e9
    e["source"] = f"{rep} (ncu --set full --clock-control none, {'c3' if NX == 2048 else 'c2'} interior chunk, tools/profile_kernels.py)"
    return {k: e[k] for k in ("kernel", "grid", "duration_us", "dram_bytes_per_launch", "alg_bytes_per_launch",
                              "alg_unit", "traffic_over_alg", "dram_gbs", "alg_gbs", "issue_active_pct",
                              "inst_executed", "registers", "top_stalls", "source") if k in e}


def codec_values(rep, idx=0):
    # grid (lines, arrays x row groups, slabs) since the codec kernels take the array from grid y (round 2;
    # before: grid z = arrays x slabs, grid y = row groups)
    _, gy, gz = (int(x) for x in summarise(rep)[idx]["grid"].strip("()").split(","))
    groups = (AX // 4 + 7) // 8
    planes = 4 * gz * (gy // groups)
    return planes * AX * AX, planes


if __name__ == "__main__":
    if "--c3" in sys.argv:  # a c3 interior chunk (tools/profile_kernels.py with WL=c3)
        sys.argv.remove("--c3")
        AX, NX = 2056, 2048
    if sys.argv[1] == "--chunk":
        rep = sys.argv[2]
        step, dec, enc, planes, idx = rep, rep, rep, 152, {"step": 1, "decode": 0, "encode": 5}
    else:
        step, dec, enc, planes = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
        idx = {"step": 0, "decode": 0, "encode": 0}
    out = {"step": entry(step, planes * NX * NX * 16, f"{planes} planes x {NX}^2 cell-updates x 16 B", idx["step"])}
    for name, rep in (("decode", dec), ("encode", enc)):
        v, pl = codec_values(rep, idx[name])
        out[name] = entry(rep, v * (RATE // 8 + 4), f"{pl} array-planes x {AX}^2 values x ({RATE // 8} + 4) B",
                          idx[name])
    json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
    print(json.dumps({k: {x: v.get(x) for x in ("duration_us", "traffic_over_alg", "alg_gbs", "issue_active_pct")}
                      for k, v in out.items()}, indent=1))
