"""Per-kernel table of the last N steps of an `ncu --metrics gpu__time_duration.sum --csv` launch list
(development): python tools/launch_table.py <csv> [first-kernel-of-a-step regex] [steps]."""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, ui, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value"), hdr.index("Metric Name")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
ks = [(re.sub(r"\(anonymous namespace\)::|^void ", "", r[ki].split("(")[0]), float(r[vi].replace(",", "")) * scale[r[ui]])
      for r in rows if r[mi] == "gpu__time_duration.sum"]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else "tnext_kernel")
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
starts = [i for i, k in enumerate(ks) if pat.search(k[0])]
for a, b in zip(starts[-steps:], starts[-steps + 1:] + [len(ks)]):
    print(f"--- step from launch {a}: {sum(t for _, t in ks[a:b]):.1f} us")
    for name, t in ks[a:b]:
        print(f"  {name:55s} {t:9.1f} us")
