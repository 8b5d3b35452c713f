"""Pinned D2H bandwidth of the step's result size alone vs while the C2
filter runs on another stream (is e2e bound by PCIe or by the overlap?):
python tools/probe_d2h_overlap.py"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import workload, _lib
torch.cuda.set_device(0)
v = workload.uniform_rows(0, 8, 0, 50_000_000)
lo, hi = workload.c2_queries(count=1000, levels=(1e-3,))[1e-3]
st = eng.DeviceStore(v, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE)
b = st.prepare(lo, hi, "vafile_batch")
total = b.reserve()
nbytes = total * 4
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
K = 10
def copies():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    with torch.cuda.stream(cs):
        for _ in range(K):
            dst.copy_(src, non_blocking=True)
    e1.record(cs)
    return e0, e1
for mode in ("alone", "with filter"):
    torch.cuda.synchronize()
    if mode == "with filter":
        for _ in range(K + 4):
            b.ids_async(ks.cuda_stream)
    e0, e1 = copies()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"D2H {mode}: {nbytes / ms / 1e6:.1f} GB/s ({ms:.2f} ms per {nbytes / 1e6:.0f} MB)", flush=True)
k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k0.record(ks)
for _ in range(K):
    b.ids_async(ks.cuda_stream)
k1.record(ks)
torch.cuda.synchronize()
print(f"filter+scatter alone: {k0.elapsed_time(k1) / K:.2f} ms", flush=True)
k0.record(ks)
for _ in range(K):
    b.ids_async(ks.cuda_stream)
k1.record(ks)
e0, e1 = copies()
torch.cuda.synchronize()
print(f"filter+scatter with D2H: {k0.elapsed_time(k1) / K:.2f} ms; D2H {nbytes / (e0.elapsed_time(e1) / K) / 1e6:.1f} GB/s", flush=True)
outs = [torch.empty(total + 1024, dtype=torch.int32, pin_memory=True).numpy().view("uint32") for _ in range(3)]
st.ids_stream([(lo, hi)] * 3, "vafile_batch", outs=outs)
t = time.perf_counter()
st.ids_stream([(lo, hi)] * 20, "vafile_batch", outs=[outs[k % 3] for k in range(20)])
print(f"ids_stream: {(time.perf_counter() - t) / 20 * 1e3:.2f} ms per batch", flush=True)
