"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump by CUDA source line.
usage: python scripts/ncu_lines.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, stall, inst = "?", defaultdict(float), defaultdict(float)
src = {}
hdr = None
cur_line = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur_line = (fname, int(r[0]))
        src[cur_line] = r[1]
        continue  # the CUDA line's own row repeats the sum of its SASS rows
    try:
        stall[cur_line] += float(r[4] or 0)
        inst[cur_line] += float(r[7] or 0)
    except ValueError:
        pass
ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
print(f"samples {ts:.0f}  warp-instructions {ti:.3e}")
for key in sorted(stall, key=lambda x: -stall[x])[:top]:
    print(f"{key[0]}:{key[1]:<5} stall {100*stall[key]/ts:5.1f}%  inst {100*inst[key]/ti:5.1f}%  {src[key].strip()[:90]}")
