"""Summarise an `ncu --page raw --csv` export (development): per kernel launch, duration, DRAM
bytes, achieved occupancy, issue activity and the top stall reasons (per issue-active cycle)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def num(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
print("| kernel | grid x block | regs | us | DRAM MB (r+w) | GB/s | warps active % | issue active % | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|")
for r in data:
    name = r[col["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")
    t_us = num(r, "gpu__time_duration.sum") * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units[col["gpu__time_duration.sum"]], 1.0)
    rd, wr = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum")
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    rd *= scale.get(units[col["dram__bytes_read.sum"]], 1.0)
    wr *= scale.get(units[col["dram__bytes_write.sum"]], 1.0)
    top = sorted(((num(r, s), s.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                  for s in stalls), reverse=True)[:3]
    print(f"| {name} | {r[col['Grid Size']]} x {r[col['Block Size']]} | {r[col['launch__registers_per_thread']]} | {t_us:.1f} | "
          f"{rd + wr:.1f} | {(rd + wr) / t_us * 1e3 if t_us else 0:.0f} | {num(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{num(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          + ", ".join(f"{n} {v:.2f}" for v, n in top) + " |")
