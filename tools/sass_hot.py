"""Summarise an ncu source-page SASS CSV: instructions executed by opcode and
the hottest instructions with their stall samples.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_hot.py x.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # kernel index in a multi-kernel export
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
a = starts[which]
b = starts[which + 1] if which + 1 < len(starts) else len(rows)
print("kernel:", rows[a][1][:100])
rows = rows[a:b]
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
ie = ix["Instructions Executed"]
samp = ix["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[ie] or 0) for r in body)
ops = Counter()
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += float(r[ie] or 0)
print(f"total warp instructions {tot:.4g}")
for op, c in ops.most_common(25):
    print(f"  {op:10s} {c:12.4g} {100 * c / tot:5.1f}%")
st = Counter()
for r in body:
    for h in stall_cols:
        st[h] += float(r[ix[h]] or 0)
s_all = sum(st.values())
print("stall samples:", ", ".join(f"{h[6:]} {100 * v / s_all:.1f}%" for h, v in st.most_common(8)))
print("hottest by samples:")
for r in sorted(body, key=lambda r: -float(r[samp] or 0))[:top]:
    top_st = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:2]
    print(f"  {r[ix['Address']]:>6s} {float(r[samp] or 0):7.0f} {float(r[ie] or 0):10.4g}  {r[ix['Source']][:60]:60s} {top_st}")
