"""e2e breakdown of store.ids on C2 (MDRQ_DEBUG_TIMING=1 prints phases)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=1000, levels=(1e-3,))[1e-3]
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE | _lib.LAYOUT_ROWWISE)
out = torch.empty(60_000_000, dtype=torch.int32, pin_memory=True).numpy().view("uint32")
for i in range(6):
    t = time.perf_counter()
    offs, ids = st.ids(lo, hi, out=out)
    print("wall ms", round((time.perf_counter() - t) * 1e3, 3), file=sys.stderr)
