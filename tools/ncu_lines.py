"""Per-source-line instruction / stall summary of one ncu report (ncu -i REP --page source --csv
--print-source cuda,sass): the lines that execute the most warp instructions."""
import csv, subprocess, sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, x in enumerate(rows) if "Instructions Executed" in x)
h = rows[hi]
ie, te, ss = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)")
lines = [x for x in rows[hi + 1:] if len(x) > ie and x[2] == "-"]
f = lambda s: float(s or 0)
tot = sum(f(x[ie]) for x in lines)
tots = sum(f(x[ss]) for x in lines)
print(f"total warp instructions {tot:.4g}, stall samples {tots:.0f}")
for x in sorted(lines, key=lambda x: -f(x[ie]))[:n]:
    print(f"{100 * f(x[ie]) / tot:5.1f}% inst {100 * f(x[ss]) / max(tots, 1):5.1f}% stall "
          f"thr/inst {f(x[te]) / max(f(x[ie]), 1):4.1f}  L{x[0]}: {x[1][:90]}")
