"""Single-query VA-file scan on C2 at every selectivity level (device time per
query, count and ids): python tools/probe_va_single.py [nq]"""
import sys, os
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 50
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
levels = (1e-5, 1e-4, 1e-3, 1e-2, 1e-1)
qs = workload.c2_queries(count=nq, levels=levels)
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
for s in levels:
    lo, hi = qs[s]
    out = {}
    for mode in ("count", "ids"):
        b = st.prepare(lo, hi, "vafile")
        if mode == "ids":
            b.reserve()
        b.profile(ids=(mode == "ids"))            # warm
        pr = b.profile(ids=(mode == "ids"))
        out[mode] = round(sum(x[0] for x in pr.values()) * 1e3 / nq, 1)
    print(f"vafile s={s:g} us/query count {out['count']} ids {out['ids']}", flush=True)
