"""Static SASS instruction histogram of the hot kernels in the built liboocs.so (cuobjdump -sass), the
evidence behind DESIGN.md's claims: TMA loads (UTMALDG) and mbarrier ops (SYNCS) in the stencil,
Blackwell paired fp32 (FFMA2 / FADD2 / FMUL2), three-input min/max (FMNMX3) in the encoder, the warp
transposes (SHFL, PRMT, LOP3).  Static counts (instructions in the binary, not executed ones: ncu's
inst_executed is the dynamic figure).

    python tools/sass_hist.py [--lib paper_2204_11315_b200/liboocs.so] [--out profiles/r02_sass_hist.json]
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOT = {
    "stencil_step_tma_kernel<16>": r"stencil_step_tma_kernelILi16EE",
    "star7_step_kernel": r"star7_step_kernel",
    "bq_encode_kernel<false, 15>": r"bq_encode_kernelILb0ELi15E",
    "bq_decode_kernel<false, 15>": r"bq_decode_kernelILb0ELi15E",
    "bq_encode_kernel<false, 7>": r"bq_encode_kernelILb0ELi7E",
    "bq_decode_kernel<false, 7>": r"bq_decode_kernelILb0ELi7E",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2204_11315_b200", "liboocs.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_hist.json"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            funcs[cur][m.group(1)] += 1
    out = {}
    for name, pat in HOT.items():
        hits = [f for f in funcs if re.search(pat, f)]
        if not hits:
            continue
        c = funcs[hits[0]]
        base = collections.Counter()
        for op, n in c.items():
            base[op.split(".")[0]] += n
        out[name] = {"mangled": hits[0], "total": sum(c.values()),
                     "by_opcode": dict(base.most_common()),
                     "by_opcode_with_modifiers": dict(c.most_common(40))}
    out["_source"] = f"cuobjdump -sass {os.path.relpath(a.lib, ROOT)} (static counts)"
    json.dump(out, open(a.out, "w"), indent=1)
    for k, v in out.items():
        if k.startswith("_"):
            continue
        top = ", ".join(f"{op} {n}" for op, n in list(v["by_opcode"].items())[:12])
        print(f"{k}: {v['total']} instr; {top}")


if __name__ == "__main__":
    main()
