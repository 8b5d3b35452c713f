"""Full-size configuration parity on the GPU (BASELINE.json configs C2-C5).

EVERY query of every configuration is compared with the CPU oracle: the
committed fixtures tests/golden/all_<cfg>.npz hold, per query, the oracle's
count and set hash (sum of splitmix64(id) mod 2**64; oracle/mdrq_oracle.c
oracle_hash_batch, pinned against the reference's own id lists by
tests/golden/make_all_queries.py).  The device result is checked in place
(tests/devhash.py): ids strictly ascending and < n within every query, then
(count, hash) per query == the oracle's.  That is every query on the
multi-query VA pass (what the planner runs for a batch), counts of every
query on the multi-query columnar pass, and a stratified sample of >= 500
queries on each single-query path (columnar, VA scan).

The first queries are also compared with the reference's OWN id lists
(sha1; tests/golden/c*.npz, recorded from the reference by make_golden.py).
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import golden
from devhash import batch_hashes

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


def _every_query(st, lo, hi, counts, hashes, name, single=500, single_paths=("columnar", "vafile", "columnar_batch")):
    """Every query on the planner's batch path (ids: count + hash; count
    mode: counts) and a stratified sample on the single-query paths."""
    c, h, path = batch_hashes(st, lo, hi, "auto")
    assert path == "vafile_batch", (name, path)
    assert np.array_equal(c, counts), (name, "vafile_batch counts", np.flatnonzero(c != counts)[:10])
    assert np.array_equal(h, hashes), (name, "vafile_batch ids", np.flatnonzero(h != hashes)[:10])
    assert np.array_equal(st.count(lo, hi, "vafile_batch"), counts), (name, "vafile_batch count mode")
    nq = lo.shape[0]
    k = min(nq, 1024)
    assert np.array_equal(st.count(lo[:k], hi[:k], "columnar_batch"), counts[:k]), (name, "columnar_batch")
    sel = np.unique(np.linspace(0, nq - 1, min(single, nq)).astype(np.int64))
    for p in single_paths:
        c, h, ran = batch_hashes(st, lo[sel], hi[sel], p)
        assert ran == p
        assert np.array_equal(c, counts[sel]), (name, p, "counts")
        assert np.array_equal(h, hashes[sel]), (name, p, "ids")


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
        # every query against the oracle's (count, set hash)
        A = golden(f"all_{name}.npz")
        assert np.array_equal(A["counts"], G["oracle_counts"])
        _every_query(st, lo, hi, A["counts"], A["hash"], name)


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
    SequentialScan id lists; EVERY query (10 000, 5e9 ids, checked in place)
    against the oracle's (count, set hash)."""
    from paper_1801_03644_b200 import workload
    G = golden("c5.npz")
    values = workload.c5_data()
    for s, h in zip(G["slice_starts"], G["slice_sha1"]):
        assert hashlib.sha1(values[s:s + 1_000_000].tobytes()).digest() == h.tobytes(), s
    lo, hi = workload.c5_queries()
    k = G["ref_counts"].size
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
        A = golden("all_c5.npz")
        assert np.array_equal(A["counts"][:nq], G["oracle_counts"])
        _every_query(st, lo, hi, A["counts"], A["hash"], "c5")


def test_c2_every_query_vs_oracle(c2_store):
    """C2: all 5 x 1000 queries (1e-5 .. 1e-1) against the oracle."""
    from paper_1801_03644_b200 import workload
    st, _ = c2_store
    A = golden("all_c2.npz")
    for li, (s, (lo, hi)) in enumerate(workload.c2_queries().items()):
        assert A[f"level{li}_s"][0] == s
        _every_query(st, lo, hi, A[f"level{li}_counts"], A[f"level{li}_hash"], f"c2 {s:g}", single=100)
