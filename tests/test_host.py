"""Host-side logic that needs no GPU: the boundary types (pkg/tests/test_core.py
counterparts), the generators (bit-identical to the reference's), the file
formats, and the planner-independent helpers."""

import numpy as np
import pytest

from conftest import golden
from paper_1801_03644_b200 import (
    DataSet,
    GeneratorSpec,
    KernelMode,
    RangeQuery,
    ResultSet,
    SearchStats,
    gen_uniform,
    pair_query_batch,
    read_dataset,
    read_queries,
    write_dataset,
    write_queries,
)
from paper_1801_03644_b200 import workload
from paper_1801_03644_b200.core import stack_queries
from paper_1801_03644_b200.scan import chunk_spans


class TestDataSet:
    def test_shape_and_bounds(self):
        values = np.array([[0.1, 2.0], [0.5, -1.0], [0.9, 0.0]], dtype=np.float32)
        data = DataSet(values)
        assert data.n == 3 and data.m == 2
        assert data.per_dim_bounds[0].tolist() == [np.float32(0.1), np.float32(0.9)]
        assert data.per_dim_bounds[1].tolist() == [-1.0, 2.0]

    def test_empty_allowed_zero_dims_rejected(self):
        assert DataSet(np.empty((0, 4), np.float32)).n == 0
        assert DataSet(np.empty((0, 4), np.float32)).per_dim_bounds.tolist() == [[0, 0]] * 4
        with pytest.raises(ValueError):
            DataSet(np.empty((3, 0), np.float32))

    def test_nan_rejected_and_immutable(self):
        with pytest.raises(ValueError, match="NaN"):
            DataSet(np.array([[0.1], [np.nan]], np.float32))
        data = DataSet(np.zeros((2, 2), np.float32))
        with pytest.raises(ValueError):
            data.values[0, 0] = 1.0
        with pytest.raises(AttributeError):
            data.foo = 1


class TestRangeQuery:
    def test_queried_flags_from_sentinels(self):
        q = RangeQuery([-np.inf, 0.2, -np.inf], [np.inf, 0.8, 1.0])
        assert q.queried.tolist() == [False, True, True]
        assert q.queried_dims.tolist() == [1, 2]

    def test_inverted_bounds_error(self):
        with pytest.raises(ValueError, match="dimension 1"):
            RangeQuery([0.0, 0.9], [1.0, 0.1])

    def test_point_full_domain_predicates_nan(self):
        assert RangeQuery([0.5], [0.5]).queried.tolist() == [True]
        assert not RangeQuery.full_domain(3).queried.any()
        q = RangeQuery.from_predicates(4, {1: (0.2, 0.4), 3: (0.5, 0.5)})
        assert q.queried.tolist() == [False, True, False, True]
        with pytest.raises(ValueError):
            RangeQuery.from_predicates(2, {5: (0.0, 1.0)})
        with pytest.raises(ValueError):
            RangeQuery([np.nan], [1.0])

    def test_float32_cast(self):
        q = RangeQuery([0.1], [0.3])
        assert q.lower.dtype == np.float32 and q.lower[0] == np.float32(0.1)

    def test_stack_queries(self):
        qs = [RangeQuery([0.0, 0.1], [1.0, 0.2]), RangeQuery.full_domain(2)]
        lo, hi = stack_queries(qs, 2)
        assert lo.shape == (2, 2) and lo.dtype == np.float32 and np.isneginf(lo[1]).all()
        with pytest.raises(ValueError):
            stack_queries(qs, 3)


def test_result_set_and_stats():
    rs = ResultSet.from_ids([1, 4, 9])
    rs.validate(10)
    assert len(rs) == 3 and rs == ResultSet.from_ids(np.array([1, 4, 9], np.int32))
    with pytest.raises(ValueError):
        ResultSet.from_ids([3, 2]).validate(10)
    with pytest.raises(ValueError):
        ResultSet.from_ids([10]).validate(10)
    a = SearchStats(objects_compared=3, early_breaks=1)
    a.merge(SearchStats(objects_compared=2, columns_scanned=4))
    assert (a.objects_compared, a.columns_scanned, a.early_breaks) == (5, 4, 1)
    assert KernelMode.parse("vector") is KernelMode.VECTORIZED


def test_gen_uniform_is_the_reference_generator():
    # workload.py:59-65: default_rng(seed).random((n, m), float32)
    data = gen_uniform(GeneratorSpec("uniform", 1000, 3, seed=7))
    assert np.array_equal(data.values, np.random.default_rng(7).random((1000, 3), dtype=np.float32))
    G = golden("c1.npz")
    import hashlib
    assert hashlib.sha1(workload.c1_data().tobytes()).digest() == G["data_sha1"].tobytes()


@pytest.mark.parametrize("m", [1, 3, 8, 10])
def test_uniform_rows_equals_one_shot_slices(m):
    full = np.random.default_rng(0).random((5000, m), dtype=np.float32)
    for a, b in [(0, 5000), (0, 1), (1, 2), (7, 4001), (1234, 5000), (4999, 5000), (3, 3)]:
        assert np.array_equal(workload.uniform_rows(0, m, a, b), full[a:b]), (a, b)


def test_c2_golden_data_head():
    G = golden("c2.npz")
    assert bool(G["head_equal"][0])
    assert np.array_equal(workload.c2_data(start=0, stop=1000),
                          np.random.default_rng(0).random((1000, 8), dtype=np.float32))


def test_query_generators_shapes_and_widths():
    lo, hi = workload.c1_queries()
    assert lo.shape == (1000, 3) and lo.dtype == np.float32
    assert np.allclose(hi - lo, 0.01 ** (1 / 3), atol=1e-6)
    levels = workload.c2_queries(count=10)
    assert sorted(levels) == sorted(workload.C2["levels"])
    for s, (l, h) in levels.items():
        assert np.allclose(h - l, s ** (1 / 8), atol=1e-6) and (l >= 0).all() and (h <= 1.0 + 1e-6).all()
    data = gen_uniform(GeneratorSpec("uniform", 100, 4, seed=1))
    qs = pair_query_batch(data, 5, 3)
    assert all(q.m == 4 and (q.lower <= q.upper).all() for q in qs)


def test_dataset_roundtrip(tmp_path):
    data = gen_uniform(GeneratorSpec("uniform", 37, 5, seed=2))
    p = tmp_path / "d.bin"
    write_dataset(data, p)
    back = read_dataset(p)
    assert np.array_equal(back.values, data.values)
    assert np.array_equal(read_dataset(p, mmap=True).values, data.values)
    raw = p.read_bytes()
    (tmp_path / "bad.bin").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="magic"):
        read_dataset(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="payload"):
        read_dataset(tmp_path / "short.bin")


def test_queries_jsonl_roundtrip(tmp_path):
    qs = [RangeQuery([0.1, -np.inf], [0.2, np.inf]), RangeQuery.full_domain(2)]
    p = tmp_path / "q.jsonl"
    write_queries(qs, p)
    back = read_queries(p)
    for a, b in zip(qs, back):
        assert np.array_equal(a.lower, b.lower) and np.array_equal(a.upper, b.upper)
    (tmp_path / "bad.jsonl").write_text('{"lower": [1]}\n')
    with pytest.raises(ValueError, match="bad query record"):
        read_queries(tmp_path / "bad.jsonl")


def test_chunk_spans_kat():
    # pkg/tests/test_scan.py:170-173
    assert chunk_spans(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert chunk_spans(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]


def test_methods_registry_rejects_trees_and_unknown():
    from paper_1801_03644_b200 import METHOD_NAMES, build_method
    data = DataSet(np.zeros((4, 2), np.float32))
    assert "vertical" in METHOD_NAMES and "vafile" in METHOD_NAMES
    for name in ("kdtree", "rstar", "nope"):
        with pytest.raises(ValueError):
            build_method(name, data)


def test_cli_parser_and_report_columns():
    from paper_1801_03644_b200.cli import REPORT_COLUMNS, build_parser
    # the reference's CSV header (bench.py:34-38)
    assert REPORT_COLUMNS[:3] == ("method", "n", "m") and REPORT_COLUMNS[-2:] == ("objects_compared",
                                                                                   "nodes_visited")
    a = build_parser().parse_args(["bench", "--n", "10", "--queries", "3", "--out", "x.csv"])
    assert (a.cmd, a.n, a.count, a.out) == ("bench", 10, 3, "x.csv")


def _lop3(a, b, c, lut):
    """PTX lop3.b32: bit i of the result = bit (a_i << 2 | b_i << 1 | c_i) of lut."""
    r = np.zeros_like(a)
    for mt in range(8):
        if (lut >> mt) & 1:
            ta = a if mt & 4 else ~a
            tb = b if mt & 2 else ~b
            tc = c if mt & 1 else ~c
            r |= ta & tb & tc
    return r


def test_va_swar_range_test_exhaustive():
    """numpy restatement of vafile.cu swar_range / swar_and (the single-query
    VA filter's byte-code range test, LOP3 tables as in the kernel), checked
    for every code byte in every byte position against every code range
    0 <= lo <= hi <= 255 and the empty encodings (lo > hi, lo = 256, hi = -1)."""
    H = np.uint32(0x80808080)
    v = np.arange(256, dtype=np.uint32)
    words = [v << np.uint32(8 * p) | (np.uint32(0x5A) << np.uint32(8 * ((p + 1) & 3))) for p in range(4)]
    ranges = [(lo, hi) for lo in range(256) for hi in range(lo, 256)] + [(5, 4), (256, 0), (0, -1), (256, 255)]
    for lo, hi in ranges:
        empty = lo > hi or lo > 255 or hi < 0
        l = 0 if empty else lo
        w = 0 if empty else hi - lo
        c1 = np.uint32((l * 0x01010101) & 0x7F7F7F7F)
        km = np.uint32(0 if l & 0x80 else 0xFFFFFFFF)
        wH = np.uint32((w * 0x01010101) | 0x80808080)
        wm = np.uint32(0xFFFFFFFF if w & 0x80 else 0)
        live = np.uint32(0 if empty else 0xFFFFFFFF)
        for p, x in enumerate(words):
            b = (x | H) - c1
            t = wH - (b & ~H)
            d = _lop3(b, x, np.full_like(x, km), 0x96)
            le = _lop3(d, np.full_like(x, wm), t, 0x8E)
            got = (_lop3(np.full_like(x, H), le, np.full_like(x, live), 0x80) >> np.uint32(8 * p + 7)) & 1
            want = np.zeros(256, np.uint32) if empty else ((v >= lo) & (v <= hi)).astype(np.uint32)
            assert np.array_equal(got, want), (lo, hi, p)
    # flags_to_nib: bits 7, 15, 23, 31 -> bits 0..3
    f = np.arange(16, dtype=np.uint32)
    flags = sum(((f >> np.uint32(i)) & 1) << np.uint32(8 * i + 7) for i in range(4))
    nib = ((((flags >> np.uint32(7)) & np.uint32(0x01010101)) * np.uint32(0x00204081)) >> np.uint32(21)) & 15
    assert np.array_equal(nib, f)


def test_verify_ground_truth_on_cpu():
    """cli.ground_truth: the reference's SequentialScan(SCALAR) when the
    reference is importable (baseline/_ref), else numpy containment; both
    equal the C oracle's ids (no device involved)."""
    import os
    import oracle
    from paper_1801_03644_b200.cli import ground_truth
    from paper_1801_03644_b200.workload import GeneratorSpec, gen_dataset, pair_query_batch
    from conftest import ROOT
    data = gen_dataset(GeneratorSpec("uniform", 5000, 4, seed=3))
    queries = pair_query_batch(data, 20, 4)
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/nonexistent"):
        exp, src = ground_truth(data, queries, path)
        for q, e in zip(queries, exp):
            assert np.array_equal(e, oracle.brute_ids(data.values, q.lower, q.upper)), src
