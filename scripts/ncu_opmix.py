"""Opcode mix (executed warp-instructions per SASS opcode) from an ncu source-page CSV dump
(`ncu -i rep --page source --csv --print-source cuda,sass`).  usage: ncu_opmix.py dump.csv [units]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 0
op = collections.Counter(); seen = set(); tot = 0
for r in rows:
    if len(r) < 9 or r[0] or r[2] in ("-", "...", "Address") or not r[2].startswith("0x"):
        continue
    if r[2] in seen:  # a SASS row listed under several source lines
        continue
    seen.add(r[2])
    try:
        n = float(r[7] or 0)
    except ValueError:
        continue
    t = r[3].split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    op[o.split(".")[0]] += n
    tot += n
print(f"total warp-instructions {tot:.4g}" + (f"  ({tot * 32 / units:.2f} thread-instructions per unit)" if units else ""))
for o, n in op.most_common(40):
    print(f"{o:12s} {100 * n / tot:5.1f}%" + (f"  {n * 32 / units:6.2f} per unit" if units else ""))
