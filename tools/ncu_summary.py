"""Summarise ncu --set full reports (gpurun_out/*.ncu-rep) into JSON: per kernel duration, DRAM bytes,
achieved GB/s, issue activity and the top stall reasons."""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
}
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3,
         "us": 1, "ms": 1e3, "ns": 1e-3, "Ghz": 1e3, "Mhz": 1, "hz": 1e-6}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "")[:80], "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for k, m in KEYS.items():
            if m in d:
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                e[k] = v * UNITS.get(u.get(m, ""), 1)
        stalls = {h.split("issue_stalled_")[1].split("_per_issue")[0]: float(d[h]) for h in hdr
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                  and d.get(h, "").replace(".", "").isdigit()}
        e["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        if "dram_read_bytes" in e and "duration_us" in e:
            e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
            e["dram_gbs"] = e["dram_bytes"] / (e["duration_us"] * 1e-6) / 1e9
        res.append(e)
    return res


if __name__ == "__main__":
    print(json.dumps({rep: summarise(rep) for rep in sys.argv[1:]}, indent=1))
