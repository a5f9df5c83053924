"""Per-source-line totals of an `ncu --page source --csv --print-source sass` export (development):
python tools/ncu_lines.py <sass.csv> <nvdisasm -g output> <mangled kernel name> <source.cu> [top]
Maps the i-th SASS row of the export to the i-th instruction of the kernel in the line-annotated
disassembly and sums executed instructions and warp-stall samples per source line."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > ss]
lines, cur, inside = [], None, False
for ln in open(sys.argv[2]):
    if ln.startswith(".text.") or ln.startswith("\t.text."):
        inside = sys.argv[3] in ln and ln.strip().endswith(":")
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*", line (\d+)', ln)
    if m:
        cur = int(m.group(1))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", ln):
        lines.append(cur)
print(f"sass rows {len(body)}, disassembled instructions {len(lines)}")
src = open(sys.argv[4]).read().split("\n")
inst, samp = collections.Counter(), collections.Counter()
for r, l in zip(body, lines):
    inst[l] += int(r[ie] or 0)
    samp[l] += int(r[ss] or 0)
ti, ts = sum(inst.values()), sum(samp.values())
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
print(f"instructions {ti:.3e}, samples {ts}")
for l, _ in sorted(samp.items(), key=lambda kv: -kv[1])[:top]:
    text = src[l - 1].strip()[:90] if l else "?"
    print(f"{l!s:>5} inst {100 * inst[l] / ti:5.1f}%  samples {100 * samp[l] / ts:5.1f}%  {text}")
