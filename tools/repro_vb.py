"""Small vafile_batch ids repro vs the oracle: python tools/repro_vb.py n m nq s"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1801_03644_b200 as eng
n, m, nq, s = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
rng = np.random.default_rng(1)
v = rng.random((n, m), dtype=np.float32)
w = s ** (1 / m)
lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
hi = (lo + w).astype(np.float32)
ec = oracle.count_batch(v, lo, hi)
eo, ei = oracle.ids_batch(v, lo, hi, counts=ec)
with eng.DeviceStore(v, layouts=1 | 4) as st:
    c = st.count(lo, hi, "vafile_batch")
    print("count ok", np.array_equal(c, ec))
    o, i = st.ids(lo, hi, "vafile_batch")
    print("ids ok", np.array_equal(o, eo) and np.array_equal(i.astype(np.int64), ei), int(eo[-1]))
