"""Hottest SASS lines of an `ncu --page source --csv --print-source sass` export (development):
python tools/ncu_hot_sass.py <csv> [top] -> samples, share, instruction, with +-3 lines of context."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, ai = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
body = [r for r in rows[2:] if len(r) > si]
samples = [int(r[si] or 0) for r in body]
tot = sum(samples)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total samples {tot}")
order = sorted(range(len(body)), key=lambda i: -samples[i])[:top]
for i in sorted(order):
    print(f"{i:6d} {samples[i]:7d} {100 * samples[i] / tot:5.1f}%  {body[i][ai].strip()}")
