"""One prepared batch of a configuration, for ncu captures and quick probes.

    PROF_CFG=c5 PROF_PATH=vafile_batch PROF_NQ=10000 PROF_MODE=both python tools/prof_c5.py
    ncu --set full -k regex:va_batch_kernel -s 3 -c 2 python tools/prof_c5.py

PROF_CFG: c5 (5e8 x 10, the bench workload) or c2 (5e7 x 8, 1e-3); PROF_PATH:
any path name; PROF_NQ: queries of the batch; PROF_MODE: count / ids / both
(each after one untimed sizing run, reserve(), which runs the ids pass once).
Prints the device time of each timed pass (CUDA events on the launching
stream) so a plain run doubles as a probe.
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
    cfg = os.environ.get("PROF_CFG", "c5")
    nq = int(os.environ.get("PROF_NQ", "1024"))
    path = os.environ.get("PROF_PATH", "vafile_batch")
    mode = os.environ.get("PROF_MODE", "both")
    reps = int(os.environ.get("PROF_REPS", "1"))
    t = time.time()
    if cfg == "c2":
        values = workload.c2_data()
        lo, hi = workload.c2_queries(count=nq, levels=(1e-3,))[1e-3]
    else:
        values = workload.c5_data(workers=os.cpu_count())
        lo, hi = workload.c5_queries(count=nq)
    layouts = _lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE | (_lib.LAYOUT_ROWWISE if path == "rowwise" else 0)
    st = eng.DeviceStore(values, layouts=layouts, va_bits=8)
    del values
    b = st.prepare(lo, hi, path)
    total = b.reserve()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    torch.cuda.synchronize()
    print(f"setup {time.time() - t:.1f}s info {b.info()} ids {total}", flush=True)
    for m in (("count", "ids") if mode == "both" else (mode,)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push(m)   # ncu --nvtx --nvtx-include "<mode>/" selects these launches
        e0.record(stream)
        for _ in range(reps):
            if m == "count":
                b.count_async(0, sp)
            else:
                b.ids_async(sp)
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print(f"{m}: {e0.elapsed_time(e1) / reps:.3f} ms per batch", flush=True)
    b.close()
    st.close()


if __name__ == "__main__":
    main()
