"""Per-phase device cost of the bit-sliced pass on one configuration (count
and ids, filter / id write split): python tools/probe_cfg.py c3 [path]"""
import os
import sys
sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_1801_03644_b200 as eng
from paper_1801_03644_b200 import _lib
from bench_configs import load


def main():
    cfg = sys.argv[1]
    path = sys.argv[2] if len(sys.argv) > 2 else "vafile_batch"
    values, lo, hi, desc = load(cfg)
    nq = lo.shape[0]
    st = eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    stream = torch.cuda.Stream()
    b = st.prepare(lo, hi, path)
    row = {"info": b.info()}
    for mode in ("count", "ids"):
        if mode == "ids":
            b.reserve()
        pr = b.profile(ids=(mode == "ids"), stream=stream.cuda_stream)
        row[mode] = {k: round(v[0] * 1e3 / nq, 2) for k, v in pr.items()}
    print(cfg, os.environ.get("MDRQ_VB_WORDS", "4"), row, flush=True)


if __name__ == "__main__":
    main()
