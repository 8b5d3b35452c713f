"""Wall time of one-query calls through the public API on C2 (host overhead
vs device time): python tools/probe_single.py"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=200, levels=(1e-3,))[1e-3]
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
for path in ("vafile", "columnar"):
    for mode in ("count", "ids"):
        f = (lambda i: st.count(lo[i:i + 1], hi[i:i + 1], path)) if mode == "count" else \
            (lambda i: st.ids(lo[i:i + 1], hi[i:i + 1], path))
        for i in range(5):
            f(i)
        t = time.perf_counter()
        for i in range(100):
            f(i)
        dt = (time.perf_counter() - t) / 100
        print(path, mode, "wall us per call", round(dt * 1e6, 1), flush=True)
# the reference-API method objects
data = eng.DataSet(v)
for name in ("gpu_vafile", "gpu_columnar"):
    m = eng.build_method(name, data)
    qs = [eng.RangeQuery(lo[i], hi[i]) for i in range(100)]
    for q in qs[:5]:
        m.search(q)
    t = time.perf_counter()
    for q in qs:
        m.search(q)
    print(name, "search() wall us", round((time.perf_counter() - t) / len(qs) * 1e6, 1), flush=True)
    m.close()
