"""Probe one path on C2: python tools/probe_path.py <path> <mode> [nq]"""
import sys, os
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
path, mode = sys.argv[1], sys.argv[2]
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 5
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=nq, levels=(1e-3,))[1e-3]
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE | _lib.LAYOUT_ROWWISE)
b = st.prepare(lo, hi, path)
if mode == "ids":
    b.reserve()
pr = b.profile(ids=(mode == "ids"))
print(path, mode, {k: (round(v[0] * 1e3 / nq, 3), v[1]) for k, v in pr.items()}, "us/query")
