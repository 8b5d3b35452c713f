"""Access-method parity on the GPU (pkg/tests/test_scan.py, test_vafile.py
counterparts): every GPU path returns the oracle's id set for every query."""

import hashlib

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu

PATHS = ("columnar", "rowwise", "vafile", "columnar_batch", "vafile_batch")
ALL_LAYOUTS = 1 | 2 | 4


def sha1_ids(ids):
    return hashlib.sha1(np.ascontiguousarray(ids, dtype="<u4").tobytes()).digest()


def check_store(gpu, values, lo, hi, paths=PATHS, va_bits=8):
    lo = np.ascontiguousarray(lo, np.float32).reshape(-1, values.shape[1])
    hi = np.ascontiguousarray(hi, np.float32).reshape(-1, values.shape[1])
    exp_counts = oracle.count_batch(values, lo, hi)
    exp_offs, exp_ids = oracle.ids_batch(values, lo, hi, counts=exp_counts)
    with gpu.DeviceStore(values, layouts=ALL_LAYOUTS, va_bits=va_bits) as st_:
        for p in paths:
            counts = st_.count(lo, hi, p)
            assert np.array_equal(counts, exp_counts), p
            offs, ids = st_.ids(lo, hi, p)
            assert np.array_equal(offs, exp_offs), p
            assert np.array_equal(ids.astype(np.int64), exp_ids), p


# -- reference KATs (test_scan.py:32-45, test_core.py:83-86) -------------------

def test_enumerated_example(gpu):
    data = gpu.DataSet(np.array([[0.1], [0.5], [0.9]], dtype=np.float32))
    for name in ("sequential", "vertical", "horizontal", "vafile"):
        m = gpu.build_method(name, data, threads=2)
        assert m.search(gpu.RangeQuery([0.2], [0.9])).ids.tolist() == [1, 2], name
        m.close()


def test_full_domain_and_empty_interval(gpu):
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 50, 3, seed=1))
    for name in ("sequential", "vertical", "horizontal", "vafile"):
        m = gpu.build_method(name, data, threads=2)
        assert m.search(gpu.RangeQuery.full_domain(3)).ids.tolist() == list(range(50)), name
        assert len(m.search(gpu.RangeQuery([-5.0, 0.0, 0.0], [-1.0, 1.0, 1.0]))) == 0, name
        m.close()


def test_boundary_inclusive(gpu):
    data = gpu.DataSet(np.array([[0.25], [0.9], [0.2499], [0.9001]], np.float32))
    for name in ("sequential", "vertical", "vafile"):
        m = gpu.build_method(name, data)
        assert m.search(gpu.RangeQuery([0.25], [0.9])).ids.tolist() == [0, 1], name
        m.close()


def test_dimension_mismatch(gpu):
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 10, 2, seed=1))
    for name in ("sequential", "vertical", "vafile"):
        m = gpu.build_method(name, data)
        with pytest.raises(ValueError):
            m.search(gpu.RangeQuery([0.0], [1.0]))
        m.close()


def test_vertical_stats_and_zero_dims(gpu):
    # test_scan.py:105-121
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 300, 19, seed=3))
    vs = gpu.VerticalScan(data, threads=2)
    q = gpu.RangeQuery.from_predicates(19, {2: (0.1, 0.9), 7: (0.2, 0.8), 11: (0.0, 1.0)})
    rs, st = vs.search_with_stats(q)
    assert st.columns_scanned == 3 and st.objects_compared == 900
    assert rs.ids.tolist() == oracle.brute_ids(data.values, q.lower, q.upper).tolist()
    rs, st = vs.search_with_stats(gpu.RangeQuery.full_domain(19))
    assert rs.ids.tolist() == list(range(300)) and st.columns_scanned == 0
    vs.close()


def test_sequential_stats_early_breaks(gpu):
    rng = np.random.default_rng(4)
    v = rng.random((5000, 9), dtype=np.float32)
    data = gpu.DataSet(v)
    lo = np.full(9, 0.2, np.float32)
    hi = np.full(9, 0.9, np.float32)
    for mode, code in ((gpu.KernelMode.SCALAR, 0), (gpu.KernelMode.VECTORIZED, 1)):
        s = gpu.SequentialScan(data, mode)
        rs, st = s.search_with_stats(gpu.RangeQuery(lo, hi))
        exp_ids, n, early = oracle.scan_rows(v, lo, hi, code)
        assert np.array_equal(rs.ids, exp_ids) and st.objects_compared == n and st.early_breaks == early
        s.close()


# -- golden edge cases -------------------------------------------------------

def test_edge_values_vs_reference_golden(gpu):
    E = golden("edge.npz")
    values = E["values"]
    offs = np.concatenate([[0], np.cumsum(E["counts"])])
    with gpu.DeviceStore(values, layouts=ALL_LAYOUTS, va_bits=2) as st_:
        for p in PATHS:
            o, ids = st_.ids(E["lo"], E["hi"], p)
            assert np.array_equal(o, offs), p
            assert np.array_equal(ids.astype(np.int64), E["ids"]), p
    cat = E["cat_values"]
    for bits in (1, 3, 8):
        with gpu.DeviceStore(cat, layouts=ALL_LAYOUTS, va_bits=bits) as st_:
            for p in PATHS:
                o, ids = st_.ids(E["cat_lo"], E["cat_hi"], p)
                assert np.array_equal(np.diff(o), E["cat_counts"]), (p, bits)
                for i in range(E["cat_lo"].shape[0]):
                    assert sha1_ids(ids[o[i]:o[i + 1]]) == E["cat_sha1"][i].tobytes(), (p, bits, i)


@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 8191, 8193, 70001])
def test_ragged_sizes(gpu, n):
    rng = np.random.default_rng(n)
    m = 5
    v = rng.random((n, m), dtype=np.float32)
    lo = (rng.random((7, m)) * 0.5).astype(np.float32)
    hi = lo + np.float32(0.55)
    lo[0] = -np.inf
    hi[0] = np.inf       # full domain -> all ids
    check_store(gpu, v, lo, hi)


@pytest.mark.parametrize("m", [1, 2, 3, 7, 8, 9, 16, 19, 33, 64, 65, 100, 256])
def test_dimensionalities(gpu, m):
    rng = np.random.default_rng(100 + m)
    n = 20000
    v = rng.random((n, m), dtype=np.float32)
    k = min(m, 6)
    lo = np.full((40, m), -np.inf, np.float32)
    hi = np.full((40, m), np.inf, np.float32)
    w = 0.05 ** (1.0 / k)
    for q in range(40):
        dims = rng.choice(m, size=int(rng.integers(1, k + 1)), replace=False)
        a = rng.random(dims.size) * (1 - w)
        lo[q, dims] = a
        hi[q, dims] = a + w
    check_store(gpu, v, lo, hi)


@given(seed=st.integers(0, 2**20), n=st.integers(1, 30000), m=st.integers(1, 20), bits=st.integers(1, 8))
@settings(max_examples=25, deadline=None)
def test_random_partial_match_vs_oracle(gpu, seed, n, m, bits):
    rng = np.random.default_rng(seed)
    v = rng.random((n, m), dtype=np.float32)
    if rng.random() < 0.3:   # low-cardinality columns -> duplicate quantile boundaries
        v = np.floor(v * 4) / 4
    nq = int(rng.integers(1, 40))
    lo = np.full((nq, m), -np.inf, np.float32)
    hi = np.full((nq, m), np.inf, np.float32)
    for q in range(nq):
        dims = rng.choice(m, size=int(rng.integers(0, m + 1)), replace=False)
        a, b = np.sort(rng.random((2, dims.size)), axis=0)
        lo[q, dims] = a
        hi[q, dims] = b
        if rng.random() < 0.2 and dims.size:   # point predicate on an existing value
            j = dims[0]
            lo[q, j] = hi[q, j] = v[int(rng.integers(0, n)), j]
    check_store(gpu, v, lo, hi, va_bits=bits)


def test_methods_agree_on_pair_queries(gpu):
    # test_scan.py:199-208 / test_acceptance.py:63-92 analogue
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 10_000, 5, seed=1))
    queries = gpu.pair_query_batch(data, 200, seed=4)
    expected = [oracle.brute_ids(data.values, q.lower, q.upper) for q in queries]
    for name in ("sequential", "horizontal", "vertical", "vafile"):
        m = gpu.build_method(name, data, threads=2, seed=5)
        for q, exp in zip(queries, expected):
            assert np.array_equal(m.search(q).ids, exp), name
        br = m.search_batch(queries)
        for i, exp in enumerate(expected):
            assert np.array_equal(br[i].ids, exp), name
        assert np.array_equal(m.count_batch(queries), [e.size for e in expected]), name
        m.close()


def test_selectivity_oracle_gpu(gpu):
    data = gpu.DataSet(np.array([[0.1], [0.5], [0.9]], dtype=np.float32))
    st = gpu.selectivity_oracle(data, gpu.RangeQuery([0.2], [0.9]))
    assert st.joint == pytest.approx(2 / 3) and st.per_dim[0] == pytest.approx(2 / 3)
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 2000, 4, seed=5))
    q = gpu.RangeQuery.from_predicates(4, {1: (0.2, 0.7), 3: (0.1, 0.3)})
    st = gpu.selectivity_oracle(data, q)
    v = data.values
    assert st.per_dim[0] == 1.0 and st.per_dim[2] == 1.0
    assert st.per_dim[1] == np.count_nonzero((v[:, 1] >= np.float32(0.2)) & (v[:, 1] <= np.float32(0.7))) / 2000
    assert st.joint == oracle.brute_ids(v, q.lower, q.upper).size / 2000


def test_vafile_grid_and_soundness(gpu):
    data = gpu.gen_uniform(gpu.GeneratorSpec("uniform", 50_000, 3, seed=16))
    va = gpu.VaFile.from_dataset(data, bits=4)
    b = va.grid.boundaries
    assert b.shape == (3, 15) and np.all(np.diff(b, axis=1) >= 0)
    # equal-frequency cells on uniform data: each holds ~1/16 of the tuples
    cells = va.grid.approximate_all(data.values)[:, 0]
    frac = np.bincount(cells, minlength=16) / data.n
    assert np.all(np.abs(frac - 1 / 16) < 0.01)
    for q in gpu.pair_query_batch(data, 20, 17):
        rs, stt = va.search_with_stats(q)
        assert np.array_equal(rs.ids, oracle.brute_ids(data.values, q.lower, q.upper))
        assert stt.columns_scanned == 3
    va.close()


def test_c1_all_queries_vs_reference_golden(gpu):
    """C1: all 1000 queries, every path, ids identical to the reference's
    SequentialScan (sha1 of each id list recorded from the reference)."""
    from paper_1801_03644_b200 import workload
    G = golden("c1.npz")
    values = workload.c1_data()
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes()
    lo, hi = workload.c1_queries()
    with gpu.DeviceStore(values, layouts=ALL_LAYOUTS, va_bits=8) as st_:
        for p in PATHS:
            assert np.array_equal(st_.count(lo, hi, p), G["counts"]), p
            offs, ids = st_.ids(lo, hi, p)
            assert np.array_equal(np.diff(offs), G["counts"]), p
            bad = [i for i in range(lo.shape[0]) if sha1_ids(ids[offs[i]:offs[i + 1]]) != G["sha1"][i].tobytes()]
            assert not bad, (p, bad[:5])
        # partial-match queries of the reference VerticalScan
        for p in PATHS:
            offs, ids = st_.ids(G["p_lo"], G["p_hi"], p)
            assert np.array_equal(np.diff(offs), G["p_counts"]), p
            for i in range(G["p_lo"].shape[0]):
                assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G["p_sha1"][i].tobytes(), (p, i)


def test_vafile_batch_staging_overflow_and_dense_groups(gpu):
    """Single-pass ids of the bit-sliced VA batch (vabatch.cu mode 3) beyond
    its default staging pool (64K blocks x 1024 records): the pass falls back
    to the recount kernel and the pool grows, so the second call stages
    everything -- same ids both times.  Dense queries also put equal queries
    into one 32-record group of the scatter's stable ranking."""
    rng = np.random.default_rng(5)
    n, m, nfull = 1_200_000, 3, 60
    values = rng.random((n, m), dtype=np.float32)
    lo = np.full((nfull + 4, m), -np.inf, np.float32)
    hi = np.full((nfull + 4, m), np.inf, np.float32)
    lo[nfull:] = rng.uniform(0, 0.7, (4, m)).astype(np.float32)
    hi[nfull:] = lo[nfull:] + np.float32(0.3)
    exp_counts = oracle.count_batch(values, lo[nfull:], hi[nfull:])
    exp_offs, exp_ids = oracle.ids_batch(values, lo[nfull:], hi[nfull:], counts=exp_counts)
    every = np.arange(n, dtype=np.uint32)
    with gpu.DeviceStore(values, layouts=1 | 4) as st_:
        for _ in range(2):
            offs, ids = st_.ids(lo, hi, "vafile_batch")
            assert offs[nfull] == nfull * n
            for q in (0, 1, nfull // 2, nfull - 1):
                assert np.array_equal(ids[offs[q]:offs[q + 1]], every), q
            assert np.array_equal(offs[nfull:] - offs[nfull], exp_offs)
            assert np.array_equal(ids[offs[nfull]:].astype(np.int64), exp_ids)


_RECOUNT_SCRIPT = r"""
import sys
import numpy as np
import oracle
import paper_1801_03644_b200 as eng
rng = np.random.default_rng(3)
for n, m, nq, s in ((20000, 3, 5, 0.1), (300000, 8, 40, 0.01), (300000, 10, 40, 0.01), (300000, 12, 50, 0.01)):
    v = rng.random((n, m), dtype=np.float32)
    w = s ** (1 / m)
    lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
    hi = (lo + w).astype(np.float32)
    lo[0, 1:] = -np.inf
    hi[0, 1:] = np.inf
    ec = oracle.count_batch(v, lo, hi)
    eo, ei = oracle.ids_batch(v, lo, hi, counts=ec)
    with eng.DeviceStore(v, layouts=1 | 4) as st:
        o, i = st.ids(lo, hi, "vafile_batch")
        assert np.array_equal(o, eo) and np.array_equal(i.astype(np.int64), ei), (n, m, nq, s)
        for o, i in st.ids_stream([(lo, hi)] * 4, "vafile_batch"):   # the pipelined slots too
            assert np.array_equal(o, eo) and np.array_equal(i.astype(np.int64), ei), (n, m, nq, s)
print("recount ok")
"""


@pytest.mark.parametrize("cap", ["0", "3"])
def test_vafile_batch_recount_fallback(gpu, cap):
    """The recount kernel (vabatch.cu mode 2) that replaces the staged
    single pass when the staging pool overflows: the pool is capped through
    the MDRQ_VB_STAGING_BLOCKS test hook (read once per process, hence the
    subprocess), so every pass takes the fallback; ids equal the oracle's for
    narrow (staged values) and wide (global refinement) unions."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MDRQ_VB_STAGING_BLOCKS=cap, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _RECOUNT_SCRIPT], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "recount ok" in r.stdout, r.stdout + r.stderr


_WORDS_SCRIPT = r"""
import numpy as np
import oracle
import paper_1801_03644_b200 as eng
rng = np.random.default_rng(5)
# full passes (> 512 queries) over 3 / 8 / 12 / 16-dim unions: staged cells
# (<= 8 dims) and shuffled code words (wider), a dense pass (s = 0.2: steps
# that overflow the queue and drain per half sub-step), duplicates, point
# predicates, partial matches, a ragged tail
for n, m, nq, s in ((70001, 3, 600, 1e-2), (200003, 8, 1000, 1e-3), (60013, 8, 700, 0.2), (100003, 12, 700, 1e-2),
                    (50001, 16, 1024, 1e-2)):
    v = rng.random((n, m), dtype=np.float32)
    w = s ** (1 / m)
    lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
    hi = (lo + w).astype(np.float32)
    lo[1], hi[1] = lo[0], hi[0]
    lo[2, 1:], hi[2, 1:] = -np.inf, np.inf
    lo[3, 0] = hi[3, 0] = v[17, 0]
    if m > 8:
        lo[4:40, 2:], hi[4:40, 2:] = -np.inf, np.inf
    ec = oracle.count_batch(v, lo, hi)
    eo, ei = oracle.ids_batch(v, lo, hi, counts=ec)
    with eng.DeviceStore(v, layouts=1 | 4) as st:
        assert np.array_equal(st.count(lo, hi, "vafile_batch"), ec), (n, m, nq)
        o, i = st.ids(lo, hi, "vafile_batch")
        assert np.array_equal(o, eo) and np.array_equal(i.astype(np.int64), ei), (n, m, nq)
print("words ok")
"""


@pytest.mark.parametrize("words", ["1", "2", "4"])
def test_vafile_batch_word_layouts(gpu, words):
    """Every query-word layout of a full bit-sliced pass (vabatch.cu LW 32 /
    64 / 128: 1, 2 or 4 query words per lane, 1, 2 or 4 tuples per table
    load; MDRQ_VB_WORDS, read once per process, hence the subprocess) gives
    the oracle's counts and ids."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MDRQ_VB_WORDS=words, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _WORDS_SCRIPT], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "words ok" in r.stdout, r.stdout + r.stderr


def test_ids_stream_pipelined_batches(gpu):
    """DeviceStore.ids_stream (mdrq_query_ids_stream): several batches of
    different sizes and paths through the three pipelined slots (slot reuse,
    first-use pool growth, an empty batch) equal the oracle batch by batch;
    a caller buffer that is too small raises."""
    rng = np.random.default_rng(11)
    n, m = 300_000, 6
    values = rng.random((n, m), dtype=np.float32)
    batches = []
    for nq, s in ((70, 1e-2), (5, 1e-1), (0, 1e-3), (130, 1e-3), (64, 1e-2), (1, 0.5), (200, 1e-3)):
        w = s ** (1 / m)
        lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
        hi = (lo + w).astype(np.float32)
        if nq > 2:
            lo[1, 2:] = -np.inf
            hi[1, 2:] = np.inf
        batches.append((lo, hi))
    with gpu.DeviceStore(values, layouts=1 | 2 | 4) as st:
        for path in ("auto", "vafile_batch", "columnar"):
            info = {}
            res = st.ids_stream(batches, path, info=info)
            assert len(res) == len(batches) and info["h2d_bytes"] > 0
            for (lo, hi), (offs, ids) in zip(batches, res):
                if lo.shape[0] == 0:
                    assert offs.tolist() == [0] and ids.size == 0
                    continue
                ec = oracle.count_batch(values, lo, hi)
                eo, ei = oracle.ids_batch(values, lo, hi, counts=ec)
                assert np.array_equal(offs, eo) and np.array_equal(ids.astype(np.int64), ei), path
        with pytest.raises(ValueError, match="ids buffer"):
            st.ids_stream(batches[:2], "vafile_batch", outs=[np.empty(10, np.uint32)] * 2)


@pytest.mark.parametrize("pack,id_base", [("1", 0), ("1", 7 * 65536 + 4321), ("0", 0), (None, 0)])
def test_ids_stream_packed_copies(gpu, monkeypatch, pack, id_base):
    """The stream's packed device->host copies (pack.cu + mdrq_unpack_ids16):
    forced on, forced off and in the automatic mode, batches of ragged sizes
    -- empty results, one query, every tuple, lists crossing several
    65 536-id buckets -- on a store with and without an id base; every
    batch equals the oracle's ids, and mdrq_stream_info reports the copy."""
    import ctypes
    from paper_1801_03644_b200 import _lib
    if pack is None:
        monkeypatch.delenv("MDRQ_STREAM_PACK", raising=False)
    else:
        monkeypatch.setenv("MDRQ_STREAM_PACK", pack)
    monkeypatch.setenv("MDRQ_UNPACK_THREADS", "5")
    rng = np.random.default_rng(5)
    n, m = 300_001, 4
    v = rng.random((n, m), dtype=np.float32)
    batches = []
    # (2100 queries: three sorted passes, packed straight from slot order)
    for nq, w in ((40, 0.7), (1, 1.5), (300, 0.5), (17, 0.0), (1100, 0.6), (64, 0.9), (2100, 0.35), (5, 0.3)):
        lo = rng.uniform(0, max(1 - w, 1e-3), (nq, m)).astype(np.float32)
        hi = (lo + np.float32(w)).astype(np.float32)
        if w == 0.0:
            lo[:], hi[:] = 2.0, 3.0            # empty results
        if w > 1:
            lo[:], hi[:] = -np.inf, np.inf     # every tuple
        batches.append((lo, hi))
    exp = [oracle.ids_batch(v, lo, hi) for lo, hi in batches]
    with gpu.DeviceStore(v, layouts=1 | 4, va_bits=8, id_base=id_base) as st_:
        # rounds 0, 1: the steered share (the second round reuses warmed slots;
        # automatic mode packs from there); then fixed shares: every query
        # packed, a third packed and the rest raw
        for rep in range(4 if pack == "1" else 2):
            if rep >= 2:
                monkeypatch.setenv("MDRQ_STREAM_PACK_SHARE", ("1.0", "0.3")[rep - 2])
            info = {}
            outs = [np.empty(ei.size + 16, np.uint32) for _, ei in exp]
            res = st_.ids_stream(batches, "auto", outs=outs, info=info)
            for (eo, ei), (offs, ids) in zip(exp, res):
                assert np.array_equal(offs, eo)
                assert np.array_equal(ids.astype(np.int64), ei + id_base)
            out = (ctypes.c_uint64 * 4)()
            _lib.check(_lib.load().mdrq_stream_info(st_.handle, out))
            assert out[2] == len(batches)
            total = sum(int(o[-1]) for o, _ in res)
            assert info["d2h_bytes"] == out[0] and info["packed_batches"] == out[1]
            if pack == "1":
                assert out[1] == sum(1 for o, _ in res if o[-1] > 0)
                assert out[0] < 4 * total            # fewer bytes than the raw ids
            elif pack == "0":
                assert out[1] == 0
                assert out[0] >= 4 * total


@pytest.mark.parametrize("m", [3, 8, 9, 10, 11])
def test_vafile_batch_multi_pass_vs_oracle(gpu, m):
    """More queries than one bit-sliced pass holds (1 024): three passes, the
    last one partial, narrow (on-chip refinement) and wide (containment
    rows) unions, selectivities from 1e-4 to 5e-2, partial-match and point
    predicates; counts and ids equal the oracle's."""
    rng = np.random.default_rng(40 + m)
    n, nq = 200_000, 2100
    v = rng.random((n, m), dtype=np.float32)
    v[::97] = v[1::97][: v[::97].shape[0]]   # duplicate rows
    s = 10 ** rng.uniform(-4, np.log10(5e-2), nq)
    w = (s ** (1.0 / m)).astype(np.float32)[:, None]
    lo = (rng.random((nq, m)) * (1 - w)).astype(np.float32)
    hi = (lo + w).astype(np.float32)
    free = rng.random((nq, m)) < 0.25
    lo[free] = -np.inf
    hi[free] = np.inf
    pts = rng.integers(0, n, nq // 10)
    lo[: nq // 10, 0] = hi[: nq // 10, 0] = v[pts, 0]
    check_store(gpu, v, lo, hi, paths=("vafile_batch",))


@pytest.mark.parametrize("m", [4, 8, 10, 12, 13, 16])
def test_vafile_batch_code_refinement_edges(gpu, m):
    """The bit-sliced pass refines staged unions on 15-bit monotone codes
    (launch.h va_batch_q15_t: float32 values staged up to 10 dims, their
    codes above) and falls back to the float32 compare only when a code
    equals a bound's.  Data and bounds built to sit on that edge: integer
    categoricals with equality predicates, bounds one ulp either side of
    data values, a column with a huge offset (every value shares one code),
    a constant column, columns holding +-inf and +-FLT_MAX; two passes of
    full-match, partial-match and point queries against the oracle."""
    rng = np.random.default_rng(700 + m)
    n, nq = 120_000, 1100
    v = rng.random((n, m), dtype=np.float32)
    v[:, 0] = rng.integers(0, 10, n)                       # categorical
    v[:, 1] = np.float32(1e9) + rng.integers(0, 64, n) * np.float32(64)   # tiny range on a huge offset
    if m > 4:
        v[:, 2] = 7.25                                     # constant
        v[:, 3] = rng.normal(0, 1e30, n).astype(np.float32)
        v[::1001, 3] = np.inf
        v[1::1001, 3] = -np.inf
        v[2::1001, 3] = np.finfo(np.float32).max
        v[3::1001, 4] = -np.finfo(np.float32).max
    lo = np.full((nq, m), -np.inf, np.float32)
    hi = np.full((nq, m), np.inf, np.float32)
    rows = rng.integers(0, n, nq)
    for q in range(nq):
        dims = rng.choice(m, size=int(rng.integers(1, min(m, 6) + 1)), replace=False)
        for j in dims:
            a = v[rows[q], j]
            kind = rng.integers(0, 5)
            if kind == 0 or not np.isfinite(a):   # point predicate on a data value
                lo[q, j] = hi[q, j] = a
            elif kind == 1:                       # one ulp inside / outside
                lo[q, j] = np.nextafter(a, np.float32(np.inf))
                hi[q, j] = np.nextafter(v[rows[(q + 1) % nq], j], np.float32(-np.inf))
                if lo[q, j] > hi[q, j]:
                    lo[q, j], hi[q, j] = hi[q, j], lo[q, j]
            elif kind == 2:                       # a data value as the lower bound
                lo[q, j] = a
            elif kind == 3:                       # ... as the upper bound
                hi[q, j] = a
            else:
                b = v[rows[(q + 7) % nq], j]
                lo[q, j], hi[q, j] = (a, b) if a <= b else (b, a)
    check_store(gpu, v, lo, hi, paths=("vafile_batch",))


@pytest.mark.parametrize("nq", [1, 33, 200, 256, 257, 400, 512, 513])
def test_vafile_batch_lanes_per_tuple_vs_oracle(gpu, nq):
    """Passes of <= 256 / <= 512 queries pack 4 / 2 tuples per warp
    instruction (vabatch.cu LW = 8 / 16); the pass sizes around both
    thresholds, narrow (3, 8 dims) and 10-dim unions, counts and ids."""
    rng = np.random.default_rng(nq)
    n = 150_000
    for m in (3, 8, 10):
        v = rng.random((n, m), dtype=np.float32)
        s = 10 ** rng.uniform(-4, -1.3, nq)
        w = (s ** (1.0 / m)).astype(np.float32)[:, None]
        lo = (rng.random((nq, m)) * (1 - w)).astype(np.float32)
        hi = (lo + w).astype(np.float32)
        free = rng.random((nq, m)) < 0.2
        lo[free] = -np.inf
        hi[free] = np.inf
        check_store(gpu, v, lo, hi, paths=("vafile_batch",))


def test_ids64_and_bounce_buffer_paths(gpu):
    """mdrq_query_ids64 / DeviceStore.ids64 (the int64 ResultSet path of
    search()) and the pinned bounce buffer of the synchronous ids calls: a
    sequence of queries whose totals grow and shrink (speculative prefix hit,
    miss -> second copy, empty result) on every path equals ids() and the
    oracle; a result larger than the 64 MB bounce cap goes straight to the
    caller's buffer (int64: widened in place)."""
    rng = np.random.default_rng(5)
    n, m = 400_000, 4
    values = rng.random((n, m), dtype=np.float32)
    widths = (0.05, 0.9, 0.3, 1e-4, 1.0, 0.6, 0.0)
    with gpu.DeviceStore(values, layouts=ALL_LAYOUTS) as st_:
        for p in PATHS:
            for w in widths:
                lo = rng.uniform(0, 1 - w, (1, m)).astype(np.float32) if w < 1 else np.zeros((1, m), np.float32)
                hi = (lo + w).astype(np.float32)
                if w == 0.0:
                    lo[:] = 2.0
                    hi[:] = 3.0
                ec = oracle.count_batch(values, lo, hi)
                eo, ei = oracle.ids_batch(values, lo, hi, counts=ec)
                offs64, ids64 = st_.ids64(lo, hi, p)
                assert ids64.dtype == np.int64 and ids64.flags.owndata
                assert np.array_equal(offs64, eo) and np.array_equal(ids64, ei), (p, w)
                offs, ids = st_.ids(lo, hi, p)
                assert np.array_equal(offs, eo) and np.array_equal(ids.astype(np.int64), ei), (p, w)
            # a multi-query batch through ids64
            lo = rng.uniform(0, 0.5, (7, m)).astype(np.float32)
            hi = (lo + 0.5).astype(np.float32)
            ec = oracle.count_batch(values, lo, hi)
            eo, ei = oracle.ids_batch(values, lo, hi, counts=ec)
            offs64, ids64 = st_.ids64(lo, hi, p)
            assert np.array_equal(offs64, eo) and np.array_equal(ids64, ei), p
        with pytest.raises(ValueError, match="ids buffer"):
            st_.ids(np.zeros((1, m), np.float32), np.ones((1, m), np.float32), "columnar",
                    out=np.empty(10, np.uint32))
    big = 20_000_000   # 80 MB of ids > the 64 MB bounce buffer
    col = np.zeros((big, 1), np.float32)
    col[::3] = 1.0
    with gpu.DeviceStore(col, layouts=1) as st_:
        for lo_, hi_ in ((-1.0, 2.0), (0.5, 2.0), (-1.0, 2.0)):
            offs64, ids64 = st_.ids64(np.array([[lo_]], np.float32), np.array([[hi_]], np.float32), "columnar")
            want = np.arange(big, dtype=np.int64) if lo_ < 0 else np.arange(0, big, 3, dtype=np.int64)
            assert offs64.tolist() == [0, want.size] and np.array_equal(ids64, want)
        offs, ids = st_.ids(np.array([[-1.0]], np.float32), np.array([[2.0]], np.float32), "columnar")
        assert ids.size == big and ids[0] == 0 and ids[-1] == big - 1 and (np.diff(ids.astype(np.int64)) == 1).all()


def test_fetch_after_count_and_truncation(gpu):
    """A truncated ids call (ids_cap 0 -> MDRQ_ETRUNC) keeps its result for
    mdrq_fetch_ids / mdrq_fetch_ids64 even when a count call with another
    batch size runs in between (the counts reuse the pinned bounce buffer)."""
    import ctypes
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(9)
    n, m = 200_000, 3
    values = rng.random((n, m), dtype=np.float32)
    lo = rng.uniform(0, 0.6, (4, m)).astype(np.float32)
    hi = (lo + 0.4).astype(np.float32)
    ec = oracle.count_batch(values, lo, hi)
    eo, ei = oracle.ids_batch(values, lo, hi, counts=ec)
    with gpu.DeviceStore(values, layouts=ALL_LAYOUTS) as st_:
        for p in ("vafile", "columnar", "vafile_batch"):
            offs = np.zeros(5, np.uint64)
            total = ctypes.c_uint64(0)
            rc = lib.mdrq_query_ids(st_.handle, lo.ctypes.data_as(_lib.f32p), hi.ctypes.data_as(_lib.f32p), 4,
                                    _lib.PATHS[p], offs.ctypes.data_as(_lib.u64p), None, 0, ctypes.byref(total))
            assert rc == _lib.MDRQ_ETRUNC and int(total.value) == ei.size
            assert np.array_equal(offs.astype(np.int64), eo)
            c = st_.count(lo[:1], hi[:1], p)          # another batch size in between
            assert int(c[0]) == int(ec[0])
            got = np.empty(ei.size, np.uint32)
            _lib.check(lib.mdrq_fetch_ids(st_.handle, got.ctypes.data_as(_lib.u32p), got.size))
            assert np.array_equal(got.astype(np.int64), ei), p
            got64 = np.empty(ei.size, np.int64)
            _lib.check(lib.mdrq_fetch_ids64(st_.handle, got64.ctypes.data_as(_lib.i64p), got64.size))
            assert np.array_equal(got64, ei), p


@pytest.mark.parametrize("m,nq,width", [(10, 3000, 0.501), (8, 2500, 0.43), (5, 4100, 0.3), (12, 2100, 0.6)])
def test_sorted_multi_pass_batches_vs_oracle(gpu, m, nq, width):
    """Batches of several 1024-query passes: the host sorts the queries into
    passes (band-sparse cell masks) and the kernel skips pruned tuples; the
    ids come back in the batch's query order.  Every query is compared with
    the oracle (count + set hash), also with a share of partial-match,
    empty and unconstrained queries in the batch."""
    from devhash import batch_hashes
    rng = np.random.default_rng(m * 1000 + nq)
    n = 200_003
    values = rng.random((n, m), dtype=np.float32)
    lo = rng.uniform(0, 1 - width, (nq, m)).astype(np.float32)
    hi = (lo + width).astype(np.float32)
    part = rng.random(nq) < 0.1
    free = rng.random((nq, m)) < 0.5
    lo[part[:, None] & free] = -np.inf
    hi[part[:, None] & free] = np.inf
    lo[7], hi[7] = 2.0, 3.0          # empty
    lo[11], hi[11] = -np.inf, np.inf  # every tuple
    exp_c, exp_h = oracle.hash_batch(values, lo, hi)
    with gpu.DeviceStore(values, layouts=1 | 4, va_bits=8) as st_:
        c, h, path = batch_hashes(st_, lo, hi, "vafile_batch")
        assert path == "vafile_batch"
        assert np.array_equal(c, exp_c), np.flatnonzero(c != exp_c)[:10]
        assert np.array_equal(h, exp_h), np.flatnonzero(h != exp_h)[:10]
        assert np.array_equal(st_.count(lo, hi, "vafile_batch"), exp_c)
        offs, ids = st_.ids(lo[:1500], hi[:1500], "vafile_batch")   # the synchronous path too
        assert np.array_equal(np.diff(offs), exp_c[:1500])
        assert np.array_equal(oracle.set_hash(offs, ids), exp_h[:1500])


def test_prepared_batch_lifecycle_and_async_contract(gpu):
    """a batch outliving its store is detached (destroying it
    later is safe, using it raises); ids_async refuses an unreserved batch;
    after reserve() it runs on the caller's stream and a synchronous call on
    the store's own stream right after it sees a consistent state."""
    import ctypes
    import torch
    from paper_1801_03644_b200 import _lib
    rng = np.random.default_rng(9)
    values = rng.random((50_003, 4), dtype=np.float32)
    lo = rng.uniform(0, 0.5, (40, 4)).astype(np.float32)
    hi = (lo + 0.5).astype(np.float32)
    exp_offs, exp_ids = oracle.ids_batch(values, lo, hi)
    st_ = gpu.DeviceStore(values, layouts=1 | 4, va_bits=8)
    b = st_.prepare(lo, hi, "vafile_batch")
    with pytest.raises(ValueError):
        b.ids_async(0)                      # not reserved
    assert b.reserve() == exp_offs[-1]
    s = torch.cuda.Stream()
    b.ids_async(s.cuda_stream)              # caller stream
    # a synchronous pass on the store's stream, ordered after the async one
    offs, ids = st_.ids(lo[:5], hi[:5], "columnar")
    assert np.array_equal(offs, exp_offs[:6]) and np.array_equal(ids.astype(np.int64), exp_ids[:exp_offs[5]])
    b.ids_async(s.cuda_stream)
    d_ids, d_offs, tot = b.result_device()
    s.synchronize()
    assert tot == exp_offs[-1]
    # DeviceStore.close closes its prepared batches first ...
    b2 = st_.prepare(lo, hi, "columnar_batch")
    # ... and a batch the Python side does not track (raw C handle) is
    # detached by mdrq_store_destroy: destroying it afterwards is safe
    lib = _lib.load()
    raw = ctypes.c_void_p()
    f32p = ctypes.POINTER(ctypes.c_float)
    lo_c, hi_c = np.ascontiguousarray(lo), np.ascontiguousarray(hi)
    _lib.check(lib.mdrq_batch_prepare(st_.handle, lo_c.ctypes.data_as(f32p), hi_c.ctypes.data_as(f32p),
                                      lo.shape[0], _lib.PATHS["vafile_batch"], ctypes.byref(raw)))
    st_.close()
    assert b2._h is None
    assert lib.mdrq_batch_destroy(raw) == 0


def test_store_bounds_for_every_layout(gpu):
    """DeviceStore.bounds() is the observed per-dim [min, max]
    (core.py:99-105) for a row-wise-only store too."""
    rng = np.random.default_rng(4)
    values = (rng.random((10_007, 6), dtype=np.float32) * 5 - 2).astype(np.float32)
    exp = np.stack([values.min(0), values.max(0)], 1)
    for layouts in (1, 2, 4, 2 | 4):
        with gpu.DeviceStore(values, layouts=layouts, va_bits=8) as st_:
            assert np.array_equal(st_.bounds(), exp), layouts


def test_reference_api_batches_use_the_multi_query_passes(gpu):
    """VaFile.search_batch / count_batch go through the planner
    (the bit-sliced pass from 10 queries); VerticalScan.search_batch through
    the multi-query columnar pass; results equal the oracle."""
    from paper_1801_03644_b200 import workload
    rng = np.random.default_rng(12)
    values = rng.random((30_011, 5), dtype=np.float32)
    lo = rng.uniform(0, 0.6, (50, 5)).astype(np.float32)
    hi = (lo + 0.4).astype(np.float32)
    queries = workload.queries_from_arrays(lo, hi)
    exp_offs, exp_ids = oracle.ids_batch(values, lo, hi)
    data = gpu.DataSet(values)
    for name in ("vafile", "vertical"):
        m = gpu.build_method(name, data)
        try:
            res = m.search_batch(queries)
            assert np.array_equal(res.offsets, exp_offs), name
            assert np.array_equal(res.ids.astype(np.int64), exp_ids), name
            assert np.array_equal(m.count_batch(queries), np.diff(exp_offs)), name
            # the batch ran the multi-query path the planner picks
            b = m.store.prepare(lo, hi, "auto")
            assert b.info()["path"] == ("vafile_batch" if name == "vafile" else "columnar_batch"), name
            b.close()
            streamed = m.search_stream([queries, queries[:7]])
            assert np.array_equal(streamed[0].offsets, exp_offs)
            assert np.array_equal(streamed[1].ids.astype(np.int64), exp_ids[:exp_offs[7]])
        finally:
            m.close()


def test_planner_batches_when_the_rows_pay(gpu):
    """MDRQ_PATH_AUTO on a VA-file store (store.cu resolve_path): the
    bit-sliced pass when the queries' dims sum to >= 10x the union's dims (and
    there are >= 10 queries), else one VA scan per query -- full-match
    batches from 10 queries on, sparse partial-match batches later; either
    way the ids are the oracle's."""
    rng = np.random.default_rng(77)
    n, m = 60_000, 12
    v = rng.random((n, m), dtype=np.float32)

    def batch(nq, k):
        lo = np.full((nq, m), -np.inf, np.float32)
        hi = np.full((nq, m), np.inf, np.float32)
        for q in range(nq):
            dims = rng.choice(m, size=k, replace=False)
            a = rng.random(k) * 0.5
            lo[q, dims] = a
            hi[q, dims] = a + 0.5
        return lo, hi

    with gpu.DeviceStore(v, layouts=1 | 4, va_bits=8) as st_:
        for nq, k, want in ((9, 12, "vafile"), (10, 12, "vafile_batch"), (16, 2, "vafile"),
                            (59, 2, "vafile"), (64, 2, "vafile_batch"), (1024, 1, "vafile_batch")):
            lo, hi = batch(nq, k)
            b = st_.prepare(lo, hi, "auto")
            assert b.info()["path"] == want, (nq, k, b.info())
            b.close()
            eo, ei = oracle.ids_batch(v, lo, hi)
            offs, ids = st_.ids(lo, hi, "auto")
            assert np.array_equal(offs, eo) and np.array_equal(ids.astype(np.int64), ei), (nq, k)
