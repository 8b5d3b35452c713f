"""Probe: event-timed pass vs mdrq_batch_profile for the single-query paths."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=100, levels=(1e-3,))[1e-3]
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); sp = s.cuda_stream
for path in ("columnar", "vafile"):
    b = st.prepare(lo, hi, path); b.reserve()
    for mode in ("count", "ids"):
        run = (lambda: b.ids_async(sp)) if mode == "ids" else (lambda: b.count_async(0, sp))
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); run(); run(); e1.record(s); torch.cuda.synchronize()
        ev = e0.elapsed_time(e1) / 2 / 100 * 1e3
        t0 = time.perf_counter(); run(); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) / 100 * 1e6
        pr = b.profile(ids=(mode == "ids"), stream=sp)
        print(f"{path:9s} {mode:5s} events {ev:7.1f} us/q  wall {wall:7.1f} us/q  profile {pr}", flush=True)
