"""Every-query fixtures for the full-size configurations (C2-C5).

    python tests/golden/make_all_queries.py [c2 c3 c4 c5]

For EVERY query of a configuration this records the oracle's result as
(count, set hash): ``hash = sum of splitmix64(id) mod 2**64`` over the
query's matching ids (oracle/mdrq_oracle.c ``oracle_hash_batch``, the
reference's ``_match_code`` predicate, _kernels_cy.pyx:23-46, applied
row by row like SequentialScan, scan.py:103-111).  The GPU tests check that
the device's ids are strictly ascending and then compare (count, hash) per
query, which pins the id list itself (a sorted duplicate-free list is fixed
by its set).

The oracle is pinned here before anything is written, against the
reference's own results recorded by make_golden.py: every reference id list
in c2/c3/c4/c5.npz (sha1) is re-derived from ``oracle.ids_batch`` on the same
rows, and its set hash must equal ``hash_batch``'s; every count in those
files (reference and pinned-oracle counts) must match.

Runs on CPU in the build container (OpenMP over the host cores: C5, 5e12
(row, query) pairs, takes ~20-30 min on 8 cores).  Writes
tests/golden/all_<cfg>.npz.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1801_03644_b200 import workload  # noqa: E402


def _sha1(ids):
    return hashlib.sha1(np.ascontiguousarray(ids, dtype="<u4").tobytes()).digest()


def _pin(values, lo, hi, ref_counts, ref_sha1, counts, hashes, id0=0):
    """The reference's id lists (sha1) for queries [0, k) against the oracle's
    ids, and the oracle's ids against hash_batch."""
    k = ref_counts.size
    offs, ids = oracle.ids_batch(values, lo[:k], hi[:k])
    ids = ids + id0
    assert np.array_equal(np.diff(offs), ref_counts), "oracle ids_batch vs reference counts"
    for i in range(k):
        assert _sha1(ids[offs[i]:offs[i + 1]]) == ref_sha1[i].tobytes(), f"reference id list {i}"
    assert np.array_equal(counts[:k], ref_counts), "hash_batch counts vs reference"
    assert np.array_equal(hashes[:k], oracle.set_hash(offs, ids)), "hash_batch hash vs oracle ids"


def make_c2():
    G = np.load(os.path.join(HERE, "c2.npz"))
    values = workload.c2_data()
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes()
    out = {}
    for li, (s, (lo, hi)) in enumerate(workload.c2_queries().items()):
        t = time.time()
        c, h = oracle.hash_batch(values, lo, hi)
        _pin(values, lo, hi, G[f"level{li}_counts"], G[f"level{li}_sha1"], c, h)
        out[f"level{li}_s"] = np.array([s])
        out[f"level{li}_counts"] = c
        out[f"level{li}_hash"] = h
        print(f"c2 level {s:g}: {time.time() - t:.0f} s, mean count {c.mean():.1f}", flush=True)
    return out


def make_generated(name, data_fn):
    G = np.load(os.path.join(HERE, f"{name}.npz"))
    values = data_fn()
    assert hashlib.sha1(values.tobytes()).digest() == G["data_sha1"].tobytes(), "generator drifted"
    lo, hi = G["lo"], G["hi"]
    t = time.time()
    c, h = oracle.hash_batch(values, lo, hi)
    assert np.array_equal(c, G["oracle_counts"]), f"{name}: counts vs the pinned oracle"
    _pin(values, lo, hi, G["ref_counts"], G["ref_sha1"], c, h)
    print(f"{name}: {time.time() - t:.0f} s, mean count {c.mean():.1f}", flush=True)
    return {"counts": c, "hash": h}


def make_c5(chunk_rows=1 << 25):
    G = np.load(os.path.join(HERE, "c5.npz"))
    lo, hi = workload.c5_queries()
    n = workload.C5["n"]
    counts = np.zeros(lo.shape[0], np.int64)
    hashes = np.zeros(lo.shape[0], np.uint64)
    k = G["ref_counts"].size
    ref_offs = [np.zeros(1, np.int64)]
    ref_ids = []
    t = time.time()
    slices = dict(zip(G["slice_starts"].tolist(), G["slice_sha1"]))
    for start in range(0, n, chunk_rows):
        stop = min(n, start + chunk_rows)
        values = workload.c5_data(start, stop)
        for s, sh in slices.items():
            if start <= s and s + 1_000_000 <= stop:
                assert hashlib.sha1(values[s - start:s - start + 1_000_000].tobytes()).digest() == sh.tobytes()
        oracle.hash_batch(values, lo, hi, id0=start, counts=counts, hashes=hashes)
        o, ids = oracle.ids_batch(values, lo[:k], hi[:k])
        ref_offs.append(np.diff(o))
        ref_ids.append((o, ids + start))
        del values
        print(f"c5 rows {stop}/{n}: {time.time() - t:.0f} s", flush=True)
    assert np.array_equal(counts[:G["oracle_counts"].size], G["oracle_counts"]), "c5 counts vs pinned oracle"
    # stitch the first k queries' ids across chunks, then pin against the reference
    per_q = [np.concatenate([ids[o[i]:o[i + 1]] for o, ids in ref_ids]) for i in range(k)]
    assert np.array_equal(np.array([p.size for p in per_q]), G["ref_counts"]), "c5 reference counts"
    for i in range(k):
        assert _sha1(per_q[i]) == G["ref_sha1"][i].tobytes(), f"c5 reference id list {i}"
        assert int(oracle.id_hash(per_q[i]).sum(dtype=np.uint64)) == int(hashes[i]), f"c5 hash {i}"
    return {"counts": counts, "hash": hashes}


def main(argv):
    cfgs = argv or ["c4", "c2", "c3", "c5"]
    for cfg in cfgs:
        if cfg == "c2":
            out = make_c2()
        elif cfg == "c3":
            out = make_generated("c3", workload.c3_data)
        elif cfg == "c4":
            out = make_generated("c4", workload.c4_data)
        elif cfg == "c5":
            out = make_c5()
        else:
            raise SystemExit(f"unknown config {cfg}")
        np.savez_compressed(os.path.join(HERE, f"all_{cfg}.npz"), **out)
        print(f"wrote all_{cfg}.npz", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
