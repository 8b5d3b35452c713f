"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Three layers must agree: the golden vectors recorded from the reference
(tests/golden/*.npz, made by tests/golden/make_golden.py), the C
restatement (oracle/mdrq_oracle.c) and the numpy restatements; and, when
oracle/_ref was built, the reference's own compiled kernels.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import golden


def sha1_ids(ids):
    return hashlib.sha1(np.ascontiguousarray(ids, dtype="<u4").tobytes()).digest()


@pytest.fixture(scope="module")
def K():
    return golden("kernels.npz")


@pytest.mark.parametrize("m", [1, 7, 8, 9, 20, 100])
def test_match_row_vs_reference_golden(K, m):
    rows, lo, hi = K[f"match_m{m}_row"], K[f"match_m{m}_lo"], K[f"match_m{m}_hi"]
    for i in range(rows.shape[0]):
        assert oracle.match_row(rows[i], lo[i], hi[i], 0) == K[f"match_m{m}_scalar"][i]
        assert oracle.match_row(rows[i], lo[i], hi[i], 1) == K[f"match_m{m}_blocked"][i]
        # pkg/tests/test_kernels.py:18-19 naive oracle
        naive = all(a <= v <= b for v, a, b in zip(rows[i].tolist(), lo[i].tolist(), hi[i].tolist()))
        assert naive == K[f"match_m{m}_scalar"][i]


def test_scan_rows_vs_reference_golden(K):
    for ci, (n, m) in enumerate(K["scan_cases"]):
        v, lo, hi = K[f"scan{ci}_values"], K[f"scan{ci}_lo"], K[f"scan{ci}_hi"]
        ids_s, cmp_s, early_s = oracle.scan_rows(v, lo, hi, 0)
        ids_b, _, early_b = oracle.scan_rows(v, lo, hi, 1)
        assert np.array_equal(ids_s, K[f"scan{ci}_ids"])
        assert np.array_equal(ids_b, K[f"scan{ci}_ids"])
        assert cmp_s == n
        assert [early_s, early_b] == K[f"scan{ci}_early"].tolist()
        assert np.array_equal(oracle.brute_ids(v, lo, hi), K[f"scan{ci}_ids"])


def test_scan_column_vs_reference_golden(K):
    for ci, n in enumerate(K["col_cases"]):
        col = K[f"col{ci}_col"]
        lo, hi = K[f"col{ci}_lohi"]
        expected = K[f"col{ci}_mask"]
        assert np.array_equal(oracle.scan_column(col, lo, hi), expected)
        assert np.array_equal(oracle.packbits_mask(col, lo, hi), expected)


def test_early_break_counter_kat():
    # pkg/tests/test_kernels.py:89-97
    values = np.array([[0.5, 0.5], [2.0, 0.5], [0.5, 2.0]], dtype=np.float32)
    ids, compared, early = oracle.scan_rows(values, np.zeros(2), np.ones(2), 0)
    assert ids.tolist() == [0] and compared == 3 and early == 1


def test_mask_helpers_kats():
    # pkg/tests/test_scan.py:97-103, 170-173
    m1 = np.packbits([1, 1, 0, 0], bitorder="little")
    m2 = np.packbits([1, 0, 1, 0], bitorder="little")
    merged = oracle.and_masks([m1, m2])
    assert np.unpackbits(merged, count=4, bitorder="little").tolist() == [1, 0, 0, 0]
    assert np.array_equal(oracle.and_masks_chunked([m1, m2], 2), merged)
    assert oracle.chunk_spans(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert oracle.chunk_spans(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    rng = np.random.default_rng(3)
    mask = rng.integers(0, 256, 37, dtype=np.uint8)
    assert oracle.mask_popcount(mask) == int(np.unpackbits(mask).sum())
    assert np.array_equal(oracle.mask_to_ids(mask, 290), oracle.np_mask_to_ids(mask, 290))


def test_edge_cases_vs_reference_golden():
    E = golden("edge.npz")
    values = E["values"]
    off = 0
    for i in range(E["lo"].shape[0]):
        c = int(E["counts"][i])
        exp = E["ids"][off:off + c]
        off += c
        ids, _, _ = oracle.scan_rows(values, E["lo"][i], E["hi"][i], 0)
        assert np.array_equal(ids, exp), i
        assert np.array_equal(oracle.brute_ids(values, E["lo"][i], E["hi"][i]), exp), i
    cat = E["cat_values"]
    offs, ids = oracle.ids_batch(cat, E["cat_lo"], E["cat_hi"], threads=2)
    assert np.array_equal(np.diff(offs), E["cat_counts"])
    for i in range(E["cat_lo"].shape[0]):
        assert sha1_ids(ids[offs[i]:offs[i + 1]]) == E["cat_sha1"][i].tobytes(), i


def test_c1_batch_oracle_vs_reference_golden():
    """All 1000 C1 queries: the OpenMP batch oracle reproduces the reference's
    SequentialScan counts and id lists (sha1)."""
    from paper_1801_03644_b200 import workload
    G = golden("c1.npz")
    values = workload.c1_data()
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes()
    lo, hi = workload.c1_queries()
    counts = oracle.count_batch(values, lo, hi)
    assert np.array_equal(counts, G["counts"])
    offs, ids = oracle.ids_batch(values, lo[:50], hi[:50], counts=counts[:50])
    for i in range(50):
        assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G["sha1"][i].tobytes(), i
    first = G["first_ids"]
    assert np.array_equal(ids[:first.size], first)


def test_c1_partial_match_vs_reference_golden():
    from paper_1801_03644_b200 import workload
    G = golden("c1.npz")
    values = workload.c1_data()
    counts = oracle.count_batch(values, G["p_lo"], G["p_hi"])
    assert np.array_equal(counts, G["p_counts"])


def test_va_code_is_count_of_boundaries_le():
    b = np.array([0.1, 0.2, 0.2, 0.5], np.float32)
    for v, c in [(-1.0, 0), (0.1, 1), (0.15, 1), (0.2, 3), (0.49, 3), (0.5, 4), (9.0, 4)]:
        assert oracle.va_code(b, v) == c
        assert int(np.searchsorted(b, np.float32(v), side="right")) == c
    col = np.random.default_rng(0).random(1000, dtype=np.float32)
    assert np.array_equal(oracle.va_encode(col, b), np.searchsorted(b, col, side="right").astype(np.uint8))


def test_reference_build_matches_restatement():
    """oracle/_ref (the reference's own compiled kernels) agrees with the C
    restatement -- skipped where the reference build is absent."""
    ref = oracle.load_reference_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    assert ref.BACKEND == "compiled"
    rng = np.random.default_rng(5)
    for m in (1, 3, 8, 9, 19):
        v = rng.random((5000, m), dtype=np.float32)
        lo = (rng.random(m) * 0.5).astype(np.float32)
        hi = lo + np.float32(0.6)
        for mode in (0, 1):
            a = ref.scan_rows(v, lo, hi, mode)
            b = oracle.scan_rows(v, lo, hi, mode)
            assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]


def test_reference_horizontal_scan_matches_oracle():
    rng = np.random.default_rng(9)
    v = rng.random((20000, 5), dtype=np.float32)
    scan = oracle.ReferenceHorizontalScan(v, threads=3, seed=4)
    try:
        for _ in range(5):
            lo = (rng.random(5) * 0.5).astype(np.float32)
            hi = lo + np.float32(0.5)
            assert np.array_equal(scan.search(lo, hi), oracle.brute_ids(v, lo, hi))
    finally:
        scan.close()


# -- the every-query checker (oracle_hash_batch) ---------------------------------

def test_hash_batch_vs_reference_c1_all_queries():
    """oracle.hash_batch against the reference's own id lists: for all 1000
    C1 queries the reference-pinned ids (sha1 vs the reference for 1000 of
    them) hash to hash_batch's value, and the counts agree; C1 partial-match
    counts too (the +-inf sentinel dims are skipped by hash_batch)."""
    from paper_1801_03644_b200 import workload
    G = golden("c1.npz")
    values = workload.c1_data()
    lo, hi = workload.c1_queries()
    c, h = oracle.hash_batch(values, lo, hi)
    assert np.array_equal(c, G["counts"])
    offs, ids = oracle.ids_batch(values, lo, hi, counts=c)
    for i in range(lo.shape[0]):
        assert sha1_ids(ids[offs[i]:offs[i + 1]]) == G["sha1"][i].tobytes(), i
    assert np.array_equal(h, oracle.set_hash(offs, ids))
    pc, _ = oracle.hash_batch(values, G["p_lo"], G["p_hi"])
    assert np.array_equal(pc, G["p_counts"])


def test_hash_batch_chunked_and_edges():
    """Streaming in row chunks with id offsets equals one call; ragged tails,
    empty results, all-unconstrained queries, +-inf / -0.0 / subnormal values
    (the edge goldens' data) agree with the scalar restatement."""
    E = golden("edge.npz")
    rng = np.random.default_rng(3)
    v = rng.random((30_011, 6), dtype=np.float32)
    v[::97, 2] = -0.0
    v[5::101, 3] = np.float32(1e-45)
    lo = rng.uniform(0, 0.5, (33, 6)).astype(np.float32)
    hi = (lo + 0.5).astype(np.float32)
    lo[0] = 2.0
    hi[0] = 3.0                                # empty
    lo[1], hi[1] = -np.inf, np.inf             # every row
    lo[2, 2], hi[2, 2] = 0.0, 0.0              # -0.0 == 0.0
    offs, ids = oracle.ids_batch(v, lo, hi)
    c, h = oracle.hash_batch(v, lo, hi)
    assert np.array_equal(c, np.diff(offs)) and np.array_equal(h, oracle.set_hash(offs, ids))
    c2 = np.zeros_like(c)
    h2 = np.zeros_like(h)
    for s in range(0, v.shape[0], 7_000):
        oracle.hash_batch(v[s:s + 7_000], lo, hi, id0=s, counts=c2, hashes=h2)
    assert np.array_equal(c2, c) and np.array_equal(h2, h)
    for pre in ("", "cat_"):   # the reference-recorded edge cases
        vals, el, eh = E[pre + "values"], E[pre + "lo"], E[pre + "hi"]
        o, i = oracle.ids_batch(vals, el, eh)
        cc, hh = oracle.hash_batch(vals, el, eh)
        assert np.array_equal(cc, E[pre + "counts"]), pre
        assert np.array_equal(cc, np.diff(o)) and np.array_equal(hh, oracle.set_hash(o, i)), pre


def test_hash_batch_rejects_nan():
    v = np.zeros((10, 2), np.float32)
    v[3, 1] = np.nan
    with pytest.raises(ValueError):
        oracle.hash_batch(v, np.zeros((1, 2), np.float32), np.ones((1, 2), np.float32))


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_every_query_fixtures_consistent(cfg):
    """The committed every-query fixtures agree with the earlier pinned
    counts (reference counts and oracle counts in c*.npz)."""
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, f"all_{cfg}.npz")
    if not os.path.exists(path):
        pytest.skip(f"all_{cfg}.npz not generated")
    A, G = golden(f"all_{cfg}.npz"), golden(f"{cfg}.npz")
    if cfg == "c2":
        for li in range(5):
            k = G[f"level{li}_counts"].size
            assert A[f"level{li}_counts"].size == 1000 and A[f"level{li}_hash"].dtype == np.uint64
            assert np.array_equal(A[f"level{li}_counts"][:k], G[f"level{li}_counts"])
    else:
        assert A["hash"].dtype == np.uint64 and A["counts"].size == A["hash"].size
        assert np.array_equal(A["counts"][:G["ref_counts"].size], G["ref_counts"])
        assert np.array_equal(A["counts"][:G["oracle_counts"].size], G["oracle_counts"])
