"""Row partitioning and multi-GPU fan-out / fan-in.

Reference: /root/reference/pkg/src/mdrq/parallel.py -- a seeded random
layout of p near-equal row partitions (make_layout, parallel.py:98-118),
one worker task per partition (WorkerPool, parallel.py:45-78) and a
concatenate + sort merge (PartitionedIndex, parallel.py:126-167).

On B200 the partitions are GPUs, one process per GPU:

* rows are split into CONTIGUOUS shards ``[r*ceil(n/W), ...)`` (``shard_range``)
  so a shard's local id + its start is the global id and rank-order
  concatenation is already sorted (no sort);
* each rank scans its shard with the device kernels;
* counts are combined with one all_gather; ids with an all_gather of the
  per-query counts followed by an all_gather of the (padded) id buffers and a
  vectorised scatter into rank order.  Over NCCL this runs on NVLink; the
  same functions run over gloo on CPU tensors for the tests.

``make_layout`` / ``PartitionLayout`` / ``WorkerPool`` keep the reference's
host-side API (HorizontalScan and build_method accept layouts).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


def default_threads() -> int:
    """MDRQ_THREADS override, else the machine's logical cores (parallel.py:20-27)."""
    env = os.environ.get("MDRQ_THREADS")
    if env:
        t = int(env)
        if t >= 1:
            return t
    return os.cpu_count() or 1


@dataclass(frozen=True)
class ExecutorConfig:
    """Worker count t; the partition count defaults to t (parallel.py:30-42)."""

    t: int

    def __post_init__(self):
        if self.t < 1:
            raise ValueError("worker count must be at least 1")

    @property
    def p(self) -> int:
        return self.t


class WorkerPool:
    """Thin reusable ThreadPoolExecutor wrapper (parallel.py:45-78)."""

    def __init__(self, workers: int):
        if workers < 1:
            raise ValueError("worker count must be at least 1")
        self.workers = workers
        self._executor: ThreadPoolExecutor | None = None

    def run(self, tasks):
        tasks = list(tasks)
        if self.workers == 1 or len(tasks) <= 1:
            return [task() for task in tasks]
        if self._executor is None:
            self._executor = ThreadPoolExecutor(max_workers=self.workers)
        futures = [self._executor.submit(task) for task in tasks]
        return [f.result() for f in futures]

    def close(self) -> None:
        if self._executor is not None:
            self._executor.shutdown(wait=True)
            self._executor = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass(frozen=True)
class PartitionLayout:
    """Balanced random assignment of n objects to p partitions (parallel.py:81-95)."""

    p: int
    seed: int
    assignment: np.ndarray
    parts: tuple

    @property
    def n(self) -> int:
        return int(self.assignment.size)

    def sizes(self) -> list[int]:
        return [int(ids.size) for ids in self.parts]


def make_layout(n: int, p: int, seed: int) -> PartitionLayout:
    """Seeded permutation split into p near-equal runs (parallel.py:98-118)."""
    if p < 1:
        raise ValueError("partition count must be at least 1")
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.int64)
    base, extra = divmod(n, p)
    parts = []
    assignment = np.empty(n, dtype=np.int32)
    start = 0
    for q in range(p):
        size = base + (1 if q < extra else 0)
        ids = perm[start:start + size]
        assignment[ids] = q
        parts.append(ids)
        start += size
    return PartitionLayout(p=p, seed=seed, assignment=assignment, parts=tuple(parts))


# ----------------------------------------------------------- GPU sharding --

def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard [start, stop) of `rank` among `world` GPUs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n // world)
    start = min(rank * per, n)
    return start, min(start + per, n)


def combine_counts(local_counts, group=None):
    """Sum per-query counts over ranks (one all_gather).  Tensor in, tensor out."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    local_counts = local_counts.to(torch.int64).contiguous().reshape(-1)
    return _all_gather(local_counts, world, group).sum(0)


def _all_gather(t, world: int, group):
    """[numel] -> [world, numel] (flat output: works on NCCL and gloo)."""
    import torch
    import torch.distributed as dist
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, t.numel())


def combine_ids(local_offsets, local_ids, group=None):
    """Rank-ordered merge of per-rank id lists.

    ``local_offsets`` int64[nq+1] and ``local_ids`` (global ids of this rank's
    shard, ascending per query) -> (offsets int64[nq+1], ids) identical on
    every rank.  Because shards are contiguous and ranks are ordered, the
    concatenation in rank order is ascending: the reference's concat + sort
    (scan.py:160, parallel.py:156-157) without the sort.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_ids.device
    local_offsets = local_offsets.to(device=dev, dtype=torch.int64)
    counts = local_offsets[1:] - local_offsets[:-1]
    nq = counts.numel()
    all_counts = _all_gather(counts.contiguous(), world, group)
    totals = all_counts.sum(1)                      # ids per rank
    per_query = all_counts.sum(0)                   # ids per query
    out_offsets = torch.zeros(nq + 1, dtype=torch.int64, device=dev)
    torch.cumsum(per_query, 0, out=out_offsets[1:])
    # rank r's segment of query q starts after ranks < r
    rank_prefix = torch.cumsum(all_counts, 0) - all_counts       # [world, nq]
    maxlen = int(totals.max().item()) if world else 0
    ids_dtype = local_ids.dtype
    padded = torch.zeros(max(maxlen, 1), dtype=ids_dtype, device=dev)
    nloc = local_ids.numel()
    if nloc:
        padded[:nloc] = local_ids
    gathered = _all_gather(padded, world, group)
    total = int(out_offsets[-1].item())
    out = torch.empty(total, dtype=ids_dtype, device=dev)
    if dev.type == "cuda" and ids_dtype.itemsize == 4:
        # one segmented-copy kernel (mdrq_copy_segments): segment (r, q) is
        # rank r's slice of query q
        import ctypes
        from . import _lib
        loff = torch.cumsum(all_counts, 1) - all_counts                 # [world, nq] within rank r
        stride = gathered.shape[1]
        src_off = (loff + torch.arange(world, device=dev, dtype=torch.int64)[:, None] * stride).contiguous()
        dst_off = (out_offsets[:-1][None, :] + rank_prefix).contiguous()
        seg_len = all_counts.contiguous()
        if total:
            _lib.check(_lib.load().mdrq_copy_segments(
                ctypes.c_void_p(gathered.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(src_off.data_ptr()), ctypes.c_void_p(dst_off.data_ptr()),
                ctypes.c_void_p(seg_len.data_ptr()), world * nq,
                ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
        return out_offsets, out
    for r in range(world):
        tr = int(totals[r].item())
        if tr == 0:
            continue
        c = all_counts[r]
        loff = torch.zeros(nq, dtype=torch.int64, device=dev)
        if nq > 1:
            torch.cumsum(c[:-1], 0, out=loff[1:])
        # destination of local element i of query q: out_off[q] + prefix[r,q] + (i - loff[q])
        base = torch.repeat_interleave(out_offsets[:-1] + rank_prefix[r] - loff, c)
        dst = base + torch.arange(tr, dtype=torch.int64, device=dev)
        out[dst] = gathered[r, :tr]
    return out_offsets, out


class ShardedScan:
    """One rank's part of a row-sharded scan over W GPUs (one process each).

    ``values`` is this rank's shard (rows [start, stop) of the dataset);
    results of ``count_batch`` / ``search_batch`` are global and identical on
    every rank.
    """

    def __init__(self, shard_values, start: int, n_total: int, *, group=None, path: str = "auto",
                 layouts=None, va_bits: int = 8, device: int | None = None):
        from . import _lib
        from .store import DeviceStore
        self.group = group
        self.start = int(start)
        self.n_total = int(n_total)
        self.path = path
        if layouts is None:
            layouts = _lib.LAYOUT_COLUMNAR
        self.store = DeviceStore(shard_values, layouts=layouts, va_bits=va_bits, device=device,
                                 id_base=self.start)
        self.m = self.store.m

    def count_batch(self, lower, upper, path: str | None = None):
        import torch
        local = self.store.count(lower, upper, path or self.path)
        dev = torch.device("cuda", self.store.device)
        return combine_counts(torch.as_tensor(local, device=dev), self.group).cpu().numpy()

    def search_batch(self, lower, upper, path: str | None = None):
        import torch
        offs, ids = self.store.ids(lower, upper, path or self.path)
        dev = torch.device("cuda", self.store.device)
        o, i = combine_ids(torch.as_tensor(offs, device=dev),
                           torch.as_tensor(ids.astype(np.int64), device=dev), self.group)
        return o.cpu().numpy(), i.cpu().numpy()

    def close(self):
        self.store.close()
