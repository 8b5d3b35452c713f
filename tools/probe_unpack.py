"""mdrq_unpack_ids16 alone on synthetic C5-shaped lists (host only): G ids/s
for thread counts and store kinds.  usage: probe_unpack.py [total_ids]"""
import ctypes
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    total = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2_000_000_000
    n, per = 500_000_000, 500_000
    nq = total // per
    nb = ((n - 1) >> 16) + 1
    offsets = (np.arange(nq + 1, dtype=np.uint64) * per)
    ids = np.empty(nq * per, np.uint32)
    base = (np.arange(per, dtype=np.int64) * 997)
    for q in range(nq):
        ids[q * per:(q + 1) * per] = (base + q * 7) % n if False else np.minimum(base + q * 7, n - 1)
    lo16 = (ids & 0xFFFF).astype(np.uint16)
    ends = np.empty((nq, nb), np.uint32)
    edges = (np.arange(1, nb + 1, dtype=np.int64) << 16)
    run0 = np.searchsorted(base, edges, side="left")
    for q in range(nq):
        ends[q] = np.searchsorted(ids[q * per:(q + 1) * per].astype(np.int64), edges, side="left") if q < 3 else \
            np.searchsorted(np.minimum(base + q * 7, n - 1), edges, side="left")
    out = np.empty(ids.size, np.uint32)
    out[:] = 0
    for T in (4, 8, 12, 16):
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            lib.mdrq_unpack_ids16(lo16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), ends.ctypes.data_as(_lib.u32p),
                                  offsets.ctypes.data_as(_lib.u64p), nq, 0, nb, out.ctypes.data_as(_lib.u32p), T)
            best = min(best, time.perf_counter() - t)
        ok = bool(np.array_equal(out, ids))
        print(f"NT={os.environ.get('MDRQ_UNPACK_NT', '1')} threads {T}: {ids.size / best / 1e9:.2f} G ids/s "
              f"({6 * ids.size / best / 1e9:.0f} GB/s) ok={ok}", flush=True)


if __name__ == "__main__":
    if "--both" in sys.argv:
        sys.argv.remove("--both")
        for nt in ("1", "0"):
            subprocess.run([sys.executable, __file__] + sys.argv[1:], env=dict(os.environ, MDRQ_UNPACK_NT=nt))
    else:
        main()
