"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of a bench command: launches per
kernel, and the kernels' shares of the last timed step (the bench's step = one oocs_run of T steps)."""
import csv
import json
import sys


def main(path, out, command, per_step=None, window=None):
    """window = "start:end" launch indices of the timed step (else the last per_step launches)."""
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    launches = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) / 1e3)
                for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    if window:
        a, b = (int(x) for x in window.split(":"))
        tail = launches[a:b]
    else:
        tail = launches[-per_step:] if per_step else launches
    share = {}
    for name, us in tail:
        base = name.split("<")[0]
        s = share.setdefault(base, {"launches": 0, "us_total": 0.0})
        s["launches"] += 1
        s["us_total"] += us
    tot = sum(s["us_total"] for s in share.values())
    for s in share.values():
        s["share"] = s["us_total"] / tot
    json.dump({"command": command, "n_launches_total": len(launches), f"timed_step_last_{len(tail)}_launches": share,
               "step_us_serialised": tot, "note": "cold-cache serialised launch times: compare shares, not absolutes",
               "launches": [[n, round(u, 3)] for n, u in launches]}, open(out, "w"), indent=0)
    print(json.dumps(share, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4] else None,
         sys.argv[5] if len(sys.argv) > 5 else None)
