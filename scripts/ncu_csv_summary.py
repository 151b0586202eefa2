"""Summarise `ncu --page raw --csv` exports (scripts/ncu_full_csv.sh) into one line per kernel."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "t_us", 1e-3), ("dram__bytes_read.sum", "dram_read_MB", 1.0),
        ("dram__bytes_write.sum", "dram_write_MB", 1.0),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1.0),
        ("smsp__inst_executed.sum", "warp_inst", 1.0),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1.0),
        ("launch__registers_per_thread", "regs", 1.0), ("launch__grid_size", "grid", 1.0),
        ("launch__block_size", "block", 1.0)]


def summarise(path):
    rows = list(csv.reader(open(path)))
    h, units, r = rows[0], rows[1], rows[2]
    out = {"kernel": r[h.index("Kernel Name")]}
    for k, name, scale in KEYS:
        if k in h:
            v = float(r[h.index(k)].replace(",", ""))
            u = units[h.index(k)]
            if name.endswith("_MB") and u == "Gbyte":
                v *= 1e3
            elif name.endswith("_MB") and u == "Kbyte":
                v *= 1e-3
            elif name.endswith("_MB") and u == "byte":
                v *= 1e-6
            if name == "t_us":
                v *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
            out[name] = round(v, 3)
    stalls = []
    for k, v in zip(h, r):
        if "smsp__average_warps_issue_stalled" in k and "per_issue_active" in k:
            try:
                stalls.append((float(v), k.split("stalled_")[1].split("_per_issue")[0]))
            except ValueError:
                pass
    out["top_stalls"] = {n: round(v, 2) for v, n in sorted(stalls, reverse=True)[:4]}
    return out


if __name__ == "__main__":
    import json
    for p in sys.argv[1:]:
        print(json.dumps(summarise(p)))
