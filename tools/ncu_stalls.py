"""Aggregate ncu source-page stall samples by opcode (and show the hottest
instructions). Usage: ncu -i rep --page source --csv --print-source sass > x.csv;
python tools/ncu_stalls.py x.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
hot = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0].split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for c in cols:
        v = int(r[ix[c]] or 0)
        by_op[op][c] += v
        tot[c] += v
    hot.append((s, src))
T = sum(tot.values())
print("total samples", T)
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:22s} {v / T:6.1%}")
print("by opcode (share of samples):")
ops = sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:12]
for op, d in ops:
    s = sum(d.values())
    top = ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:4])
    print(f"  {op:10s} {s / T:6.1%}  [{top}]")
