"""Per-kernel source-line hot spots of an ncu `--page source --csv --print-source cuda,sass`
dump holding several kernels.  usage: python scripts/ncu_funcs.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 28
func = fname = hdr = cur = None
data = defaultdict(lambda: defaultdict(lambda: [0.0, 0.0]))
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1][:48]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    try:
        data[func][cur][0] += float(r[4] or 0)
        data[func][cur][1] += float(r[7] or 0)
    except ValueError:
        pass
for f, d in data.items():
    ts = sum(v[0] for v in d.values()) or 1
    ti = sum(v[1] for v in d.values()) or 1
    print("=====", f, "inst %.3e" % ti)
    for k in sorted(d, key=lambda x: -d[x][1])[:top]:
        print(f"{k[0]}:{k[1]:<5} stall {100*d[k][0]/ts:5.1f}% inst {100*d[k][1]/ti:5.1f}%  {src[k].strip()[:80]}")
