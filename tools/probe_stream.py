"""The pipelined ids stream on the C5 bench workload with per-stage timings
(MDRQ_DEBUG_STREAM) and the host unpack alone; PROBE_NQ queries per batch."""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1801_03644_b200 as eng
    from paper_1801_03644_b200 import _lib, workload
    nq = int(os.environ.get("PROBE_NQ", "10000"))
    steps = int(os.environ.get("PROBE_STEPS", "6"))
    values = workload.c5_data(workers=os.cpu_count())
    lo, hi = workload.c5_queries(count=nq)
    st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    del values
    total = int(st.count(lo, hi).sum())
    outs = [torch.empty(total + 1024, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
    for mode in ("1", "0"):
        os.environ["MDRQ_STREAM_PACK"] = mode
        os.environ.pop("MDRQ_DEBUG_STREAM", None)
        st.ids_stream([(lo, hi)] * 3, outs=[outs[k % 2] for k in range(3)])   # warm
        os.environ["MDRQ_DEBUG_STREAM"] = "1"
        t0 = time.perf_counter()
        info = {}
        st.ids_stream([(lo, hi)] * steps, outs=[outs[k % 2] for k in range(steps)], info=info)
        dt = (time.perf_counter() - t0) / steps
        print(f"pack={mode}: {dt * 1e3:.1f} ms per step, d2h {info['d2h_bytes'] / steps / 1e9:.2f} GB per step", flush=True)
    # the host unpack alone on the last packed result
    st.close()


if __name__ == "__main__":
    main()
