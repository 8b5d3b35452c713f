"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel of the library runs at least once, and
every result is checked against the CPU oracle (so a sanitizer run is also a
parity run).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [quick]

Environment knobs the library reads once per process select the variants
(tools/gpu_sanitize.sh runs them): MDRQ_VB_WORDS=1|2|4 (query words per lane
of full bit-sliced passes), MDRQ_VB_STAGING_BLOCKS=4 (staging pool overflow:
the recount kernel, mode 2), MDRQ_VB_NO_SORT=1 (no pass sorting).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def check(st, values, lo, hi, paths):
    c_exp, h_exp = oracle.hash_batch(values, lo, hi)
    for p in paths:
        c = st.count(lo, hi, p)
        assert np.array_equal(c, c_exp), (p, "count")
        offs, ids = st.ids(lo, hi, p)
        assert np.array_equal(np.diff(offs), c_exp), (p, "ids count")
        assert np.array_equal(oracle.set_hash(offs, ids), h_exp), (p, "ids")


def boxes(rng, nq, m, width, partial=0.0):
    lo = rng.uniform(0, 1 - width, (nq, m)).astype(np.float32)
    hi = (lo + width).astype(np.float32)
    if partial:
        free = (rng.random((nq, m)) < 0.5) & (rng.random(nq) < partial)[:, None]
        lo[free], hi[free] = -np.inf, np.inf
    return lo, hi


def main():
    import paper_1801_03644_b200 as eng
    quick = "quick" in sys.argv[1:]
    rng = np.random.default_rng(11)
    n = 20_011
    cases = [(8, 300, 0.35), (8, 1000, 0.42), (10, 1000, 0.5), (5, 2100, 0.3), (10, 2100, 0.5), (20, 40, 0.85)]
    if quick:
        cases = cases[1:3] + cases[4:5]
    for m, nq, width in cases:
        values = rng.random((n, m), dtype=np.float32)
        lo, hi = boxes(rng, nq, m, width, partial=0.1)
        with eng.DeviceStore(values, layouts=1 | 2 | 4, va_bits=8, device=0) as st:
            paths = ["vafile_batch", "columnar_batch"]
            if nq <= 300:
                paths += ["columnar", "vafile", "rowwise"]
            check(st, values, lo, hi, paths)
            # the pipelined stream (copy stream + slots)
            res = st.ids_stream([(lo[:64], hi[:64])] * 3, "vafile_batch")
            c_exp, h_exp = oracle.hash_batch(values, lo[:64], hi[:64])
            for offs, ids in res:
                assert np.array_equal(oracle.set_hash(offs, ids), h_exp)
        print(f"case m={m} nq={nq}: ok", flush=True)
    # kernel-backend level (host buffers in / out)
    v = rng.random((5_003, 9), dtype=np.float32)
    lo, hi = boxes(rng, 1, 9, 0.8)
    ids, cnt, early = eng.kernels.scan_rows(v, lo[0], hi[0], 0)
    ref_ids, _, ref_early = oracle.scan_rows(v, lo[0], hi[0], 0)
    assert np.array_equal(ids, ref_ids) and early == ref_early
    mk = eng.kernels.scan_column(v[:, 0].copy(), 0.2, 0.7)
    assert np.array_equal(mk, oracle.scan_column(v[:, 0], 0.2, 0.7))
    print("kernel backend: ok", flush=True)
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
