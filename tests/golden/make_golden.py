"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the reference's
Cython kernels there (its own setup.py, ``build_ext --inplace``), imports the
reference package ``mdrq`` with ``BACKEND == "compiled"`` and records its
outputs on seeded inputs.  Nothing here is used at run time on the GPU box:
the .npz files are the committed evidence, the tests only read them.

Every expected value below comes from a reference API call:
  kernels.npz  mdrq.kernels.match_row / scan_rows / scan_column
               (_kernels_cy.pyx:49-120), both kernel modes
  edge.npz     SequentialScan(SCALAR).search on hand-built edge-case data
               (scan.py:91-114): +-inf values, -0.0, subnormals, duplicates,
               lo == hi, partial-match sentinels
  c1.npz       C1 (1e6 x 3, seed 0): SequentialScan(SCALAR) counts + sha1 of
               the id list of all 1000 queries, full ids of the first 3,
               plus 200 partial-match queries through VerticalScan
  c2.npz       C2 (5e7 x 8, seed 0): HorizontalScan (8 threads) counts +
               sha1 for the first 20 queries of each selectivity level
  c3.npz/c4.npz  C3 / C4 (our generators, workload.py): the queries, the
               reference's id lists for the first 20, oracle counts for all
  c5.npz       C5 (5e8 x 10): SequentialScan(SCALAR) id lists for the first 8
               queries, oracle counts for the first 200, table slice hashes
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

REF_PKG = "/root/reference/pkg"


def load_reference():
    scratch = os.path.join(tempfile.gettempdir(), "mdrq_ref_golden")
    if not os.path.exists(os.path.join(scratch, "setup.py")):
        shutil.rmtree(scratch, ignore_errors=True)
        shutil.copytree(REF_PKG, scratch)
    subprocess.run([sys.executable, "setup.py", "-q", "build_ext", "--inplace"], cwd=scratch, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(scratch, "src"))
    import mdrq
    assert mdrq.BACKEND == "compiled", mdrq.BACKEND
    return mdrq


def sha1_ids(ids) -> bytes:
    return hashlib.sha1(np.ascontiguousarray(ids, dtype="<u4").tobytes()).digest()


def random_case(rng, m):
    """Boundary-biased (row, lower, upper) like pkg/tests/test_kernels.py:22-40."""
    row = rng.random(m, dtype=np.float32)
    lower = rng.random(m, dtype=np.float32) - 0.5
    upper = lower + rng.random(m, dtype=np.float32)
    k = rng.integers(0, m + 1)
    contain = rng.choice(m, size=k, replace=False)
    lower[contain] = row[contain] - 0.1
    upper[contain] = row[contain] + 0.1
    if rng.random() < 0.5:
        j = rng.integers(0, m)
        lower[j] = row[j]
    if rng.random() < 0.5:
        j = rng.integers(0, m)
        upper[j] = row[j]
    upper = np.maximum(lower, upper)
    return row, lower, upper


def make_kernels(mdrq):
    k = mdrq.kernels
    out = {}
    # match_row: 300 cases per m (test_kernels.py:43-51)
    for m in (1, 7, 8, 9, 20, 100):
        rng = np.random.default_rng(1000 + m)
        rows, los, his, res_s, res_b = [], [], [], [], []
        for _ in range(300):
            r, lo, hi = random_case(rng, m)
            rows.append(r)
            los.append(lo)
            his.append(hi)
            res_s.append(k.match_row(r, lo, hi, k.MODE_SCALAR))
            res_b.append(k.match_row(r, lo, hi, k.MODE_BLOCKED))
        out[f"match_m{m}_row"] = np.stack(rows)
        out[f"match_m{m}_lo"] = np.stack(los)
        out[f"match_m{m}_hi"] = np.stack(his)
        out[f"match_m{m}_scalar"] = np.array(res_s, bool)
        out[f"match_m{m}_blocked"] = np.array(res_b, bool)
    # scan_rows: (n, m) grid with boundary rows (test_acceptance.py:95-130 style)
    cases = [(0, 3), (1, 1), (7, 2), (60, 24), (257, 5), (1000, 1), (1000, 7), (1000, 8), (1000, 9),
             (1000, 20), (1000, 100), (4099, 3), (10007, 16), (33333, 19)]
    for ci, (n, m) in enumerate(cases):
        rng = np.random.default_rng(2000 + ci)
        lower = (rng.random(m) - 0.2).astype(np.float32)
        upper = lower + (rng.random(m) * 0.8).astype(np.float32)
        values = rng.random((n, m), dtype=np.float32)
        if n:
            inside = rng.choice(n, min(n, 300), replace=False)
            values[inside] = lower + (upper - lower) * rng.random((inside.size, m), dtype=np.float32)
            edge = rng.choice(n, min(n, 100), replace=False)
            h = edge.size // 2
            values[edge[:h], rng.integers(0, m)] = lower[rng.integers(0, m)]
            values[edge[h:], rng.integers(0, m)] = upper[rng.integers(0, m)]
        ids_s, cmp_s, early_s = k.scan_rows(values, lower, upper, k.MODE_SCALAR)
        ids_b, cmp_b, early_b = k.scan_rows(values, lower, upper, k.MODE_BLOCKED)
        assert np.array_equal(ids_s, ids_b) and cmp_s == cmp_b == n
        out[f"scan{ci}_values"] = values
        out[f"scan{ci}_lo"] = lower
        out[f"scan{ci}_hi"] = upper
        out[f"scan{ci}_ids"] = ids_s
        out[f"scan{ci}_early"] = np.array([early_s, early_b], np.int64)
    out["scan_cases"] = np.array(cases, np.int64)
    # scan_column (test_kernels.py:100-113)
    for ci, n in enumerate((0, 1, 7, 8, 9, 31, 32, 33, 200, 4097)):
        rng = np.random.default_rng(3000 + ci)
        col = rng.random(n, dtype=np.float32)
        lo, hi = sorted(rng.random(2))
        out[f"col{ci}_col"] = col
        out[f"col{ci}_lohi"] = np.array([lo, hi], np.float32)
        out[f"col{ci}_mask"] = k.scan_column(col, np.float32(lo), np.float32(hi), k.MODE_BLOCKED)
    out["col_cases"] = np.array([0, 1, 7, 8, 9, 31, 32, 33, 200, 4097], np.int64)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def make_edge(mdrq):
    DataSet, RangeQuery, SequentialScan, KernelMode = (mdrq.DataSet, mdrq.RangeQuery, mdrq.SequentialScan,
                                                       mdrq.KernelMode)
    inf = np.float32(np.inf)
    sub = np.float32(1e-45)
    values = np.array([
        [0.0, -0.0, 1.0],
        [-0.0, 0.0, -1.0],
        [sub, -sub, 0.5],
        [inf, -inf, 0.25],
        [-inf, inf, 0.75],
        [0.5, 0.5, 0.5],
        [0.5, 0.5, 0.5],
        [1.0, 0.0, 0.0],
        [np.float32(3.4028235e38), np.float32(-3.4028235e38), 2.0],
        [np.float32(1.1754944e-38), 0.0, 0.5],
    ], dtype=np.float32)
    queries = [
        ([0.0, 0.0, 0.0], [0.0, 0.0, 1.0]),          # +-0 equality
        ([-0.0, -np.inf, -np.inf], [0.0, np.inf, np.inf]),
        ([0.0, -1.0, 0.0], [sub, 1.0, 1.0]),          # subnormal upper bound
        ([sub, -np.inf, -np.inf], [sub, np.inf, np.inf]),
        ([0.5, 0.5, 0.5], [0.5, 0.5, 0.5]),           # lo == hi everywhere
        ([-np.inf, -np.inf, -np.inf], [np.inf, np.inf, np.inf]),   # full domain
        ([np.inf, -np.inf, -np.inf], [np.inf, np.inf, np.inf]),    # +inf equality
        ([-np.inf, -np.inf, 0.2], [-1.0, np.inf, 0.3]),            # -inf..finite
        ([-3.4028235e38, -np.inf, -np.inf], [3.4028235e38, np.inf, np.inf]),
        ([1.0, -np.inf, -np.inf], [inf, np.inf, np.inf]),
        ([-np.inf, 0.5, -np.inf], [np.inf, 0.5, np.inf]),          # partial match
    ]
    data = DataSet(values)
    scan = SequentialScan(data, KernelMode.SCALAR)
    out = {"values": values}
    los, his, counts, ids = [], [], [], []
    for lo, hi in queries:
        q = RangeQuery(lo, hi)
        r = scan.search(q).ids
        los.append(q.lower)
        his.append(q.upper)
        counts.append(r.size)
        ids.append(r)
    out["lo"] = np.stack(los)
    out["hi"] = np.stack(his)
    out["counts"] = np.array(counts, np.int64)
    out["ids"] = np.concatenate(ids).astype(np.int64)
    # duplicates-heavy categorical data (C4-like equality predicates)
    rng = np.random.default_rng(77)
    cat = np.stack([rng.integers(0, 5, 20000).astype(np.float32),
                    rng.integers(0, 3, 20000).astype(np.float32),
                    (rng.integers(0, 2 ** 26, 20000) // 16 * 16).astype(np.float32),
                    rng.random(20000, dtype=np.float32)], axis=1)
    cdata = DataSet(cat)
    cscan = SequentialScan(cdata, KernelMode.SCALAR)
    clo, chi, ccounts, csha = [], [], [], []
    for i in range(60):
        preds = {0: (float(i % 5), float(i % 5))}
        if i % 2:
            preds[1] = (float(i % 3), float(i % 3))
        if i % 3 == 0:
            a = float(cat[i * 7, 2])
            preds[2] = (a, a + 16.0 * (i % 4) * 1e5)
        if i % 4 == 1:
            preds[3] = (0.1, 0.6)
        q = RangeQuery.from_predicates(4, preds)
        r = cscan.search(q).ids
        clo.append(q.lower)
        chi.append(q.upper)
        ccounts.append(r.size)
        csha.append(np.frombuffer(sha1_ids(r), np.uint8))
    out["cat_values"] = cat
    out["cat_lo"] = np.stack(clo)
    out["cat_hi"] = np.stack(chi)
    out["cat_counts"] = np.array(ccounts, np.int64)
    out["cat_sha1"] = np.stack(csha)
    np.savez_compressed(os.path.join(HERE, "edge.npz"), **out)


def make_c1(mdrq):
    from paper_1801_03644_b200 import workload
    values = workload.c1_data()
    ref_values = mdrq.gen_uniform(mdrq.GeneratorSpec("uniform", 1_000_000, 3, seed=0)).values
    assert np.array_equal(values, ref_values), "C1 data differs from the reference generator"
    lo, hi = workload.c1_queries()
    data = mdrq.DataSet(values)
    scan = mdrq.SequentialScan(data, mdrq.KernelMode.SCALAR)
    counts, shas, first = [], [], []
    for i in range(lo.shape[0]):
        ids = scan.search(mdrq.RangeQuery(lo[i], hi[i])).ids
        counts.append(ids.size)
        shas.append(np.frombuffer(sha1_ids(ids), np.uint8))
        if i < 3:
            first.append(ids)
    # partial-match queries through the reference VerticalScan (scan.py:167-214)
    vs = mdrq.VerticalScan(data, threads=4)
    rng = np.random.default_rng(11)
    plo, phi, pcounts, pshas, pcols = [], [], [], [], []
    for i in range(200):
        k = int(rng.integers(0, 4))  # 0..3 queried dims, 0 = full domain
        dims = rng.choice(3, size=k, replace=False)
        preds = {}
        for j in dims:
            a, b = sorted(rng.random(2))
            preds[int(j)] = (a, b)
        q = mdrq.RangeQuery.from_predicates(3, preds)
        r, st = vs.search_with_stats(q)
        plo.append(q.lower)
        phi.append(q.upper)
        pcounts.append(len(r))
        pshas.append(np.frombuffer(sha1_ids(r.ids), np.uint8))
        pcols.append(st.columns_scanned)
    vs.close()
    np.savez_compressed(
        os.path.join(HERE, "c1.npz"),
        data_sha1=np.frombuffer(hashlib.sha1(values.tobytes()).digest(), np.uint8),
        counts=np.array(counts, np.int64), sha1=np.stack(shas),
        first_ids=np.concatenate(first).astype(np.uint32),
        first_counts=np.array([a.size for a in first], np.int64),
        p_lo=np.stack(plo), p_hi=np.stack(phi), p_counts=np.array(pcounts, np.int64),
        p_sha1=np.stack(pshas), p_columns=np.array(pcols, np.int64))


def make_c2(mdrq, per_level: int = 20):
    from paper_1801_03644_b200 import workload
    values = workload.c2_data()
    head = mdrq.gen_uniform(mdrq.GeneratorSpec("uniform", 1000, 8, seed=0)).values
    data = mdrq.DataSet(values)
    scan = mdrq.build_method("horizontal", data, threads=os.cpu_count() or 8, seed=0,
                             mode=mdrq.KernelMode.SCALAR)
    out = {"data_sha1": np.frombuffer(hashlib.sha1(values.tobytes()).digest(), np.uint8),
           "head_equal": np.array([np.array_equal(values[:1000], head)])}
    for li, (s, (lo, hi)) in enumerate(workload.c2_queries().items()):
        counts, shas = [], []
        for i in range(per_level):
            ids = scan.search(mdrq.RangeQuery(lo[i], hi[i])).ids
            counts.append(ids.size)
            shas.append(np.frombuffer(sha1_ids(ids), np.uint8))
        out[f"level{li}_s"] = np.array([s])
        out[f"level{li}_counts"] = np.array(counts, np.int64)
        out[f"level{li}_sha1"] = np.stack(shas)
        print(f"  C2 level {s}: mean count {np.mean(counts):.0f}", flush=True)
    scan.close()
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **out)


def _make_generated(mdrq, name, data_fn, query_fn, ref_queries: int = 20):
    """C3 / C4: the queries themselves (slow to tune, committed), the
    reference's id lists (counts + sha1) for the first `ref_queries`, and --
    from the C oracle, which the other fixtures pin to the reference -- the
    counts of every query."""
    import oracle
    values = data_fn()
    lo, hi = query_fn()
    data = mdrq.DataSet(values)
    scan = mdrq.build_method("horizontal", data, threads=os.cpu_count() or 8, seed=0,
                             mode=mdrq.KernelMode.SCALAR)
    counts, shas = [], []
    for i in range(ref_queries):
        ids = scan.search(mdrq.RangeQuery(lo[i], hi[i])).ids
        counts.append(ids.size)
        shas.append(np.frombuffer(sha1_ids(ids), np.uint8))
    scan.close()
    all_counts = oracle.count_batch(values, lo, hi)
    assert np.array_equal(all_counts[:ref_queries], counts), "oracle disagrees with the reference"
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        data_sha1=np.frombuffer(hashlib.sha1(values.tobytes()).digest(), np.uint8),
        lo=lo, hi=hi, ref_counts=np.array(counts, np.int64), ref_sha1=np.stack(shas),
        oracle_counts=all_counts)
    print(f"  {name}: mean selectivity {all_counts.mean() / values.shape[0]:.3g}, "
          f"range {all_counts.min() / values.shape[0]:.2g}..{all_counts.max() / values.shape[0]:.2g}", flush=True)


def make_c3(mdrq):
    from paper_1801_03644_b200 import workload
    _make_generated(mdrq, "c3", workload.c3_data, workload.c3_queries)


def make_c4(mdrq):
    from paper_1801_03644_b200 import workload
    _make_generated(mdrq, "c4", workload.c4_data, workload.c4_queries)


def make_c5(mdrq, ref_queries: int = 8, oracle_queries: int = 200):
    """C5 (5e8 x 10, 20 GB): the reference's SequentialScan(SCALAR) -- the
    ground truth its own `verify` uses (cli.py:222) -- on the first
    `ref_queries` queries, the pinned C oracle's counts on the first
    `oracle_queries`, and the sha1 of 1M-row slices of the table."""
    import oracle
    from paper_1801_03644_b200 import workload
    values = workload.c5_data()
    lo, hi = workload.c5_queries()
    slices = [0, 123_456_789, 499_000_000]
    out = {"slice_starts": np.array(slices, np.int64),
           "slice_sha1": np.stack([np.frombuffer(hashlib.sha1(values[s:s + 1_000_000].tobytes()).digest(),
                                                 np.uint8) for s in slices])}
    data = mdrq.DataSet(values)
    scan = mdrq.SequentialScan(data, mdrq.KernelMode.SCALAR)
    counts, shas = [], []
    for i in range(ref_queries):
        ids = scan.search(mdrq.RangeQuery(lo[i], hi[i])).ids
        counts.append(ids.size)
        shas.append(np.frombuffer(sha1_ids(ids), np.uint8))
        print(f"  C5 query {i}: {ids.size} ids", flush=True)
    oc = oracle.count_batch(values, lo[:oracle_queries], hi[:oracle_queries])
    assert np.array_equal(oc[:ref_queries], counts), "oracle disagrees with the reference"
    out.update(ref_counts=np.array(counts, np.int64), ref_sha1=np.stack(shas), oracle_counts=oc)
    np.savez_compressed(os.path.join(HERE, "c5.npz"), **out)


def main():
    mdrq = load_reference()
    what = sys.argv[1:] or ["kernels", "edge", "c1", "c2", "c3", "c4"]
    for w in what:
        print(f"generating {w} ...", flush=True)
        {"kernels": make_kernels, "edge": make_edge, "c1": make_c1, "c2": make_c2,
         "c3": make_c3, "c4": make_c4, "c5": make_c5}[w](mdrq)
    print("done")


if __name__ == "__main__":
    main()
