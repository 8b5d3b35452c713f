"""Shared-memory wavefronts per SASS instruction from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass): totals by opcode and
every instruction above a threshold.
usage: python tools/smem_hot.py x.csv[.gz] [min_wavefronts] [kernel_index]"""
import csv
import gzip
import sys
from collections import Counter

path = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 2e7
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(fh))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
a = starts[which]
b = starts[which + 1] if which + 1 < len(starts) else len(rows)
print("kernel:", rows[a][1][:100])
hdr = rows[a + 1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[a + 2:b] if len(r) == len(hdr)]
W, WI, IE = ix["L1 Wavefronts Shared"], ix["L1 Wavefronts Shared Ideal"], ix["Instructions Executed"]
f = lambda r, k: float(r[k] or 0)
print("smem wavefronts %.4g (ideal %.4g), warp instructions %.4g" % (
    sum(f(r, W) for r in body), sum(f(r, WI) for r in body), sum(f(r, IE) for r in body)))
ops, opi, opn = Counter(), Counter(), Counter()
for r in body:
    src = r[ix["Source"]].split()
    op = src[1] if src[0].startswith("@") else src[0]
    ops[op] += f(r, W); opi[op] += f(r, WI); opn[op] += f(r, IE)
for op, c in ops.most_common(10):
    if c: print(f"  {op:22s} wavefronts {c:10.4g} ideal {opi[op]:10.4g} inst {opn[op]:10.4g} per inst {c / max(opn[op], 1):.2f}")
allops = Counter()
for r in body:
    src = r[ix["Source"]].split()
    op = src[1] if src[0].startswith("@") else src[0]
    allops[op.split(".")[0]] += f(r, IE)
print("instructions by opcode:", ", ".join(f"{o} {c:.3g}" for o, c in allops.most_common(16)))
for i, r in enumerate(body):
    if f(r, W) > thr:
        print(f"  {i:5d} {f(r, W):10.4g} ideal {f(r, WI):10.4g} inst {f(r, IE):10.4g}  {r[ix['Source']][:64]}")
