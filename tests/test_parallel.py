"""Row sharding and the multi-GPU merge, on CPU (gloo, world_size 2).

The reference's partition invariants (pkg/tests/test_parallel.py) plus the
B200 build's own: contiguous shards cover the data, and the rank-ordered
all_gather merge of per-shard id lists equals the scan of the whole table
(the reference's concat + sort, scan.py:160, without the sort)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1801_03644_b200 import make_layout
from paper_1801_03644_b200.parallel import combine_counts, combine_ids, shard_range


class TestMakeLayout:
    # pkg/tests/test_parallel.py:16-46
    def test_20_over_5_is_four_each(self):
        assert make_layout(20, 5, seed=1).sizes() == [4, 4, 4, 4, 4]

    def test_10_over_3_balanced(self):
        assert make_layout(10, 3, seed=1).sizes() == [4, 3, 3]

    def test_deterministic_and_matches_oracle_restatement(self):
        a = make_layout(100, 7, seed=42)
        b = oracle.make_layout_ids(100, 7, 42)
        for pa, pb in zip(a.parts, b):
            assert np.array_equal(pa, pb)

    def test_disjoint_and_complete(self):
        layout = make_layout(57, 4, seed=3)
        assert sorted(np.concatenate(layout.parts).tolist()) == list(range(57))
        for q, ids in enumerate(layout.parts):
            assert (layout.assignment[ids] == q).all()

    def test_more_partitions_than_objects(self):
        layout = make_layout(3, 5, seed=0)
        assert sum(layout.sizes()) == 3 and len(layout.parts) == 5

    def test_validation(self):
        with pytest.raises(ValueError):
            make_layout(10, 0, seed=0)


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (10, 3), (100, 8), (5_000_000, 8), (7, 8)])
def test_shard_range_covers_contiguously(n, world):
    spans = [shard_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(s for s in sizes if s or n < world) <= -(-n // world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, m, nq, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        values = rng.random((n, m), dtype=np.float32)
        w = 0.3 ** (1 / m)
        lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
        hi = (lo + w).astype(np.float32)
        lo[0] = -np.inf   # a full-domain query
        hi[0] = np.inf
        start, stop = shard_range(n, world, rank)
        # this rank's shard scanned by the oracle (stand-in for the device
        # scan, which needs a GPU); ids are global: local + shard start
        offs, ids = oracle.ids_batch(values[start:stop], lo, hi)
        ids = ids + start
        counts = torch.as_tensor(np.diff(offs))
        tot = combine_counts(counts)
        o, i = combine_ids(torch.as_tensor(offs), torch.as_tensor(ids))
        exp_offs, exp_ids = oracle.ids_batch(values, lo, hi)
        ok = (np.array_equal(tot.numpy(), np.diff(exp_offs)) and np.array_equal(o.numpy(), exp_offs)
              and np.array_equal(i.numpy(), exp_ids))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 20_000), (2, 1), (3, 999)])
def test_rank_ordered_merge_equals_whole_scan(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 4, 9, 7 + n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = []
    try:
        for _ in procs:
            results.append(q.get(timeout=120))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert len(results) == world and all(ok for _, ok in results), results


class _OracleShardStore:
    """The DeviceStore query interface over one row shard, answered by the
    CPU oracle (the gloo stand-in for a rank's device store; ids global)."""

    def __init__(self, values, start):
        self.values, self.start = values, start
        self.m = values.shape[1]
        self.device = 0

    def count(self, lo, hi, path="auto"):
        return oracle.count_batch(self.values, lo, hi)

    def ids(self, lo, hi, path="auto"):
        offs, ids = oracle.ids_batch(self.values, lo, hi)
        return offs, (ids + self.start).astype(np.uint32)

    def close(self):
        pass


def _sharded_worker(rank, world, port, n, m, nq, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1801_03644_b200.parallel import ShardedScan
        rng = np.random.default_rng(seed)
        values = rng.random((n, m), dtype=np.float32)
        w = 0.4 ** (1 / m)
        lo = rng.uniform(0, 1 - w, (nq, m)).astype(np.float32)
        hi = (lo + w).astype(np.float32)
        lo[1, 1:], hi[1, 1:] = -np.inf, np.inf     # partial match
        lo[2], hi[2] = 5.0, 6.0                     # empty
        start, stop = shard_range(n, world, rank)
        scan = ShardedScan(values[start:stop], start, n, store=_OracleShardStore(values[start:stop], start))
        exp_offs, exp_ids = oracle.ids_batch(values, lo, hi)
        ok = np.array_equal(scan.count_batch(lo, hi), np.diff(exp_offs))
        o, i = scan.search_batch(lo, hi)
        ok &= np.array_equal(o, exp_offs) and np.array_equal(i.astype(np.int64), exp_ids)
        # every rank writes its own slices into one node-shared host buffer
        o2, i2, buf = scan.search_batch_host(lo, hi)
        ok &= np.array_equal(o2, exp_offs) and np.array_equal(i2.astype(np.int64), exp_ids)
        del i2
        buf.close()
        q.put((rank, bool(ok)))
    except Exception as e:   # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 30_001), (3, 1_000), (2, 1)])
def test_sharded_scan_end_to_end_on_gloo(world, n):
    """ShardedScan (PartitionedIndex analog, parallel.py:126-167): counts,
    the NCCL-style merge and the direct per-rank host write all equal the
    oracle scan of the whole table."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, n, 5, 12, 11 + n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = []
    try:
        for _ in procs:
            results.append(q.get(timeout=180))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert len(results) == world and all(ok is True for _, ok in results), results
