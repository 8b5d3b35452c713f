"""Wide-union VA batch probe (C3-shaped without the generator): n x 16
uniform, 1024 partial-match queries on 2..8 random dims at ~1e-2:
python tools/probe_wide.py [n] [mode]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "count"
m, nq = 16, 1024
v = workload.uniform_rows(3, m, 0, n)
rng = np.random.default_rng(5)
lo = np.full((nq, m), -np.inf, np.float32)
hi = np.full((nq, m), np.inf, np.float32)
for q in range(nq):
    k = int(rng.integers(2, 9))
    dims = rng.choice(m, k, replace=False)
    w = 0.01 ** (1 / k)
    a = rng.uniform(0, 1 - w, k)
    lo[q, dims] = a
    hi[q, dims] = a + w
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
b = st.prepare(lo, hi, "vafile_batch")
if mode == "ids":
    b.reserve()
pr = b.profile(ids=(mode == "ids"))
print("wide", n, mode, {k: (round(x[0] * 1e3 / nq, 2), x[1]) for k, x in pr.items()}, "us/query", b.info())
