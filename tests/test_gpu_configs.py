"""Full-size configuration parity on the GPU (BASELINE.json configs).

C2 (5e7 x 8): the first 20 queries of every selectivity level against the
reference's own id lists (sha1, tests/golden/c2.npz, recorded with the
reference's HorizontalScan), and all 5000 queries through every path with
size-independent properties: count == len(ids), ids strictly ascending and
< n, and the paths agree with each other id for id.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu


def sha1_ids(ids):
    return hashlib.sha1(np.ascontiguousarray(ids, dtype="<u4").tobytes()).digest()


@pytest.fixture(scope="module")
def c2_store(gpu):
    from paper_1801_03644_b200 import workload
    values = workload.c2_data()
    G = golden("c2.npz")
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes()
    st = gpu.DeviceStore(values, layouts=1 | 2 | 4, va_bits=8)
    yield st, values
    st.close()


def test_c2_vs_reference_golden(c2_store):
    from paper_1801_03644_b200 import workload
    st, _ = c2_store
    G = golden("c2.npz")
    levels = workload.c2_queries()
    for li, (s, (lo, hi)) in enumerate(levels.items()):
        assert G[f"level{li}_s"][0] == s
        k = G[f"level{li}_counts"].size
        for path in ("columnar", "vafile", "vafile_batch", "rowwise"):
            offs, ids = st.ids(lo[:k], hi[:k], path)
            assert np.array_equal(np.diff(offs), G[f"level{li}_counts"]), (s, path)
            for i in range(k):
                assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G[f"level{li}_sha1"][i].tobytes(), (s, path, i)


def _check_generated(gpu, name, values):
    """C3 / C4: the reference's id lists for the first queries (sha1) and the
    pinned oracle's counts for every query, on the full table."""
    G = golden(f"{name}.npz")
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes(), "generator drifted"
    lo, hi = G["lo"], G["hi"]
    k = G["ref_counts"].size
    with gpu.DeviceStore(values, layouts=1 | 4, va_bits=8) as st:
        for path in ("vafile_batch", "columnar_batch", "vafile", "columnar"):
            q = lo.shape[0] if path.endswith("_batch") else 200
            assert np.array_equal(st.count(lo[:q], hi[:q], path), G["oracle_counts"][:q]), (name, path)
        for path in ("vafile_batch", "vafile", "columnar"):
            offs, ids = st.ids(lo[:k], hi[:k], path)
            assert np.array_equal(np.diff(offs), G["ref_counts"]), (name, path)
            for i in range(k):
                assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G["ref_sha1"][i].tobytes(), (name, path, i)
        # every query in ids mode: counts and cross-path id equality
        offs, ids = st.ids(lo, hi, "vafile_batch")
        assert np.array_equal(np.diff(offs), G["oracle_counts"]), name
        o2, i2 = st.ids(lo[:200], hi[:200], "columnar")
        assert np.array_equal(o2, offs[:201]) and np.array_equal(i2, ids[:o2[-1]]), name


def test_c3_vs_reference_golden(gpu):
    from paper_1801_03644_b200 import workload
    _check_generated(gpu, "c3", workload.c3_data())


def test_c4_vs_reference_golden(gpu):
    from paper_1801_03644_b200 import workload
    _check_generated(gpu, "c4", workload.c4_data())


def test_c5_full_size_vs_reference_golden(gpu):
    """C5: 5e8 x 10 (20 GB) on one GPU.  The table is generated chunk-parallel
    (PCG64 advanced per chunk) and checked against slice hashes of the
    one-shot generator; the first 8 queries against the reference's
    SequentialScan id lists, the first 200 counts against the oracle, 1024
    queries in ids mode for size-independent properties."""
    from paper_1801_03644_b200 import workload
    G = golden("c5.npz")
    values = workload.c5_data()
    for s, h in zip(G["slice_starts"], G["slice_sha1"]):
        assert hashlib.sha1(values[s:s + 1_000_000].tobytes()).digest() == h.tobytes(), s
    lo, hi = workload.c5_queries()
    k = G["ref_counts"].size
    n = values.shape[0]
    with gpu.DeviceStore(values, layouts=1 | 4, va_bits=8) as st:
        del values
        nq = G["oracle_counts"].size
        assert np.array_equal(st.count(lo[:nq], hi[:nq], "vafile_batch"), G["oracle_counts"])
        assert np.array_equal(st.count(lo[:32], hi[:32], "columnar_batch"), G["oracle_counts"][:32])
        for path in ("vafile_batch", "vafile", "columnar"):
            offs, ids = st.ids(lo[:k], hi[:k], path)
            assert np.array_equal(np.diff(offs), G["ref_counts"]), path
            for i in range(k):
                assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G["ref_sha1"][i].tobytes(), (path, i)
        offs, ids = st.ids(lo[:1024], hi[:1024], "vafile_batch")
        assert np.array_equal(np.diff(offs), st.count(lo[:1024], hi[:1024], "vafile_batch"))
        d = np.diff(ids.astype(np.int64))
        starts = offs[1:-1]
        d[starts[(starts > 0) & (starts < ids.size)] - 1] = 1
        assert (d > 0).all() and ids.max() < n


def test_c2_all_queries_paths_agree(c2_store):
    from paper_1801_03644_b200 import workload
    st, values = c2_store
    n = values.shape[0]
    for s, (lo, hi) in workload.c2_queries().items():
        ref_offs, ref_ids = st.ids(lo, hi, "vafile_batch")
        counts = np.diff(ref_offs)
        assert np.array_equal(st.count(lo, hi, "vafile_batch"), counts), s
        assert np.array_equal(st.count(lo, hi, "columnar_batch"), counts), s
        # strictly ascending within every query, all < n
        d = np.diff(ref_ids.astype(np.int64))
        starts = ref_offs[1:-1]
        d[starts[(starts > 0) & (starts < ref_ids.size)] - 1] = 1
        assert (d > 0).all() and (ref_ids.size == 0 or ref_ids.max() < n)
        sub = slice(0, 100) if s < 0.1 else slice(0, 20)   # keep the single-query paths quick
        for path in ("columnar", "vafile"):
            offs, ids = st.ids(lo[sub], hi[sub], path)
            m = offs[-1]
            assert np.array_equal(offs, ref_offs[: offs.size]), (s, path)
            assert np.array_equal(ids, ref_ids[:m]), (s, path)
        # a few queries against the OpenMP oracle on the full table
        exp = oracle.count_batch(values, lo[:4], hi[:4])
        assert np.array_equal(counts[:4], exp), s
