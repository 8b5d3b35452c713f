"""The ids stream on C2 (5e7 x 8, 1000 queries at 1e-3: 200 MB of ids per
batch), packed (automatic) against raw: ms per batch over 40 batches."""
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
    values = workload.c2_data()
    lo, hi = workload.c2_queries(levels=(1e-3,))[1e-3]
    st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    total = int(st.count(lo, hi).sum())
    outs = [torch.empty(total + 1024, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(3)]
    steps = 40
    for mode in (None, "0", "1", None):
        if mode is None:
            os.environ.pop("MDRQ_STREAM_PACK", None)
        else:
            os.environ["MDRQ_STREAM_PACK"] = mode
        st.ids_stream([(lo, hi)] * 6, outs=[outs[k % 3] for k in range(6)])
        info = {}
        t0 = time.perf_counter()
        st.ids_stream([(lo, hi)] * steps, outs=[outs[k % 3] for k in range(steps)], info=info)
        dt = (time.perf_counter() - t0) / steps
        print(f"MDRQ_STREAM_PACK={mode}: {dt * 1e3:.2f} ms per batch, packed {info['packed_batches']}/{steps}, "
              f"d2h {info['d2h_bytes'] / steps / 1e6:.0f} MB, share {info['packed_share']}", flush=True)
    st.close()


if __name__ == "__main__":
    main()
