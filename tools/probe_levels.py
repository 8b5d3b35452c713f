"""Per-selectivity-level device cost on C2 (us per query, count and ids):
python tools/probe_levels.py [paths...]"""
import sys, os
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
paths = sys.argv[1:] or ["vafile_batch", "columnar"]
v = workload.uniform_rows(0, 8, 0, 50_000_000)
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
stream = torch.cuda.Stream()
for s, (lo, hi) in workload.c2_queries().items():
    row = {}
    for p in paths:
        q = 1000 if p.endswith("_batch") else 20
        b = st.prepare(lo[:q], hi[:q], p)
        for mode in ("count", "ids"):
            if mode == "ids":
                b.reserve()
            pr = b.profile(ids=(mode == "ids"), stream=stream.cuda_stream)
            row[f"{p}.{mode}"] = round(sum(x[0] for x in pr.values()) * 1e3 / q, 2)
            if mode == "ids" and "id_write" in pr:
                row[f"{p}.ids.filter"] = round(pr["scan"][0] * 1e3 / q, 2)
                row[f"{p}.ids.write"] = round(pr["id_write"][0] * 1e3 / q, 2)
        b.close()
    print(s, row, flush=True)
