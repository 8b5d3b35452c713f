"""One C5 pass (1024 queries) in count and ids mode, for ncu captures.

    ncu --set full -k regex:va_batch_kernel -c 2 python tools/prof_c5.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1801_03644_b200 as eng
    from paper_1801_03644_b200 import _lib, workload
    nq = int(os.environ.get("PROF_NQ", "1024"))
    path = os.environ.get("PROF_PATH", "vafile_batch")
    t = time.time()
    values = workload.c5_data()
    lo, hi = workload.c5_queries(count=nq)
    st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    del values
    b = st.prepare(lo, hi, path)
    b.reserve()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    torch.cuda.synchronize()
    print(f"setup {time.time() - t:.1f}s info {b.info()}", flush=True)
    b.count_async(0, sp)
    b.ids_async(sp)
    torch.cuda.synchronize()
    print("done", flush=True)
    b.close()
    st.close()


if __name__ == "__main__":
    main()
