"""Where the wall time of one reference-API search() goes on C2 (host
phases vs device): python tools/probe_search_overhead.py"""
import sys, os, time
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
from paper_1801_03644_b200.core import stack_queries
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=200, levels=(1e-3,))[1e-3]
data = eng.DataSet(v)
m = eng.build_method("gpu_vafile", data)
qs = [eng.RangeQuery(lo[i], hi[i]) for i in range(200)]
for q in qs[:10]:
    m.search(q)
acc = {}
def tick(k, t0):
    t = time.perf_counter()
    acc[k] = acc.get(k, 0.0) + (t - t0)
    return t
N = 150
t_all = time.perf_counter()
for q in qs[10:10 + N]:
    t = time.perf_counter()
    l, h = stack_queries([q], m.m); t = tick("stack_queries", t)
    offs, ids = m.store.ids(l, h, "vafile"); t = tick("store.ids", t)
    w = m._map(ids); t = tick("_map (int64)", t)
    r = eng.ResultSet(w); t = tick("ResultSet", t)
total = time.perf_counter() - t_all
for k, s in acc.items():
    print(f"{k:16s} {s / N * 1e6:8.1f} us", flush=True)
print(f"{'total':16s} {total / N * 1e6:8.1f} us", flush=True)
t = time.perf_counter()
for q in qs[10:10 + N]:
    m.search(q)
print(f"search() {(time.perf_counter() - t) / N * 1e6:8.1f} us", flush=True)
t = time.perf_counter()
for q in qs[10:10 + N]:
    m.count(q)
print(f"count() {(time.perf_counter() - t) / N * 1e6:8.1f} us", flush=True)
os.environ["MDRQ_DEBUG_TIMING"] = "1"
