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
from paper_1801_03644_b200 import ExecutorConfig, make_layout
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
        with pytest.raises(ValueError):
            ExecutorConfig(t=0)
        assert ExecutorConfig(t=6).p == 6


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
