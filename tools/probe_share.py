"""The packed stream on the C5 bench workload at fixed packed shares and with
the steered share: ms per step over PROBE_STEPS steps (same box, same run)."""
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
    steps = int(os.environ.get("PROBE_STEPS", "14"))
    values = workload.c5_data(workers=os.cpu_count())
    lo, hi = workload.c5_queries(count=nq)
    st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    del values
    total = int(st.count(lo, hi).sum())
    outs = [torch.empty(total + 1024, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
    os.environ["MDRQ_STREAM_PACK"] = "1"
    for share in os.environ.get("PROBE_SHARES", "1.0 0.85 0.7 auto 1.0").split():
        if share == "auto":
            os.environ.pop("MDRQ_STREAM_PACK_SHARE", None)
        else:
            os.environ["MDRQ_STREAM_PACK_SHARE"] = share
        st.ids_stream([(lo, hi)] * 5, outs=[outs[k % 2] for k in range(5)])   # warm
        info = {}
        t0 = time.perf_counter()
        st.ids_stream([(lo, hi)] * steps, outs=[outs[k % 2] for k in range(steps)], info=info)
        dt = (time.perf_counter() - t0) / steps
        print(f"share {share}: {dt * 1e3:.1f} ms per step, d2h {info['d2h_bytes'] / steps / 1e9:.2f} GB per step, "
              f"share now {info['packed_share']}", flush=True)
    os.environ["MDRQ_STREAM_PACK"] = "0"
    st.ids_stream([(lo, hi)] * 3, outs=[outs[k % 2] for k in range(3)])
    t0 = time.perf_counter()
    st.ids_stream([(lo, hi)] * steps, outs=[outs[k % 2] for k in range(steps)])
    print(f"raw: {(time.perf_counter() - t0) / steps * 1e3:.1f} ms per step", flush=True)
    st.close()


if __name__ == "__main__":
    main()
