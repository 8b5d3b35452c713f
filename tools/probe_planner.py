"""Break-even of the planner's batch rule: device time of small batches
(nq queries) on the bit-sliced pass against one single-query VA scan per
query, count and ids mode, per configuration.  usage: probe_planner.py c2 c3 c4 c5"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch
    import paper_1801_03644_b200 as eng
    from paper_1801_03644_b200 import _lib
    from bench_configs import load
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    for cfg in sys.argv[1:] or ["c2"]:
        values, lo, hi, desc = load(cfg)
        st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
        del values
        rng = np.random.default_rng(0)
        pick = rng.permutation(lo.shape[0])
        for nq in (4, 8, 16, 32, 64, 128):
            l, h = lo[pick[:nq]], hi[pick[:nq]]
            kq = float(np.mean(np.sum(~(np.isneginf(l) & np.isposinf(h)), axis=1)))
            kb = int(np.sum(np.any(~(np.isneginf(l) & np.isposinf(h)), axis=0)))
            row = {"cfg": cfg, "nq": nq, "dims_per_query": round(kq, 2), "union_dims": kb}
            for path in ("vafile", "vafile_batch"):
                b = st.prepare(l, h, path)
                b.reserve()
                for mode in ("count", "ids"):
                    fn = (lambda: b.count_async(0, sp)) if mode == "count" else (lambda: b.ids_async(sp))
                    fn()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(3):
                        fn()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    row[f"{path}_{mode}_ms"] = round(e0.elapsed_time(e1) / 3, 3)
                b.close()
            print(json.dumps(row), flush=True)
        st.close()


if __name__ == "__main__":
    main()
