"""Scan-based query executors on the GPU.

Same classes, constructors and results as /root/reference/pkg/src/mdrq/scan.py:

* ``SequentialScan`` / ``HorizontalScan`` (scan.py:91-164) -> the row-wise
  kernel over a device-resident row-major store (TMA bulk-copy tiles);
* ``VerticalScan`` (scan.py:167-214) -> the fused columnar kernel: per-dim
  masks are never materialised, the AND runs in registers and the ids are
  compacted in order on the device;
* the mask helpers (scan.py:43-88) run on the GPU as well.

Every executor additionally offers ``search_batch`` / ``count`` /
``count_batch`` (the reference has no count or batch API; count is
``len(search(q))``, bench.py:176).
"""

from __future__ import annotations

import numpy as np

from . import kernels
from ._lib import MODE_BLOCKED, MODE_SCALAR
from .core import DataSet, KernelMode, RangeQuery, ResultSet, SearchStats, stack_queries
from .parallel import PartitionLayout, default_threads
from .store import DeviceStore
from . import _lib


class ColumnSet:
    """Host-side columnar view of a DataSet: m read-only float32 columns of
    one length (scan.py:17-40).  The scan itself runs on the device store's
    own ``cols[m][n_pad]`` layout; this object is the API the reference
    exposes for it."""

    __slots__ = ("columns", "n", "m")

    def __init__(self, columns):
        cols = [np.ascontiguousarray(c, dtype=np.float32) for c in columns]
        if len(cols) == 0:
            raise ValueError("at least one column required")
        length = len(cols[0]) if cols[0].ndim == 1 else -1
        if any(c.ndim != 1 or len(c) != length for c in cols):
            raise ValueError("columns must be 1-d and of equal length")
        for c in cols:
            c.setflags(write=False)
        self.columns, self.n, self.m = cols, length, len(cols)

    @classmethod
    def from_dataset(cls, data: DataSet) -> "ColumnSet":
        return cls(list(data.values.T))

    def to_matrix(self) -> np.ndarray:
        return np.stack(self.columns, axis=1)


def chunk_spans(nbytes: int, t: int) -> list[tuple[int, int]]:
    """t byte spans [start, stop) of ceil(nbytes / t) bytes, clipped at nbytes
    (so trailing spans may be empty) -- scan.py:43-52; host arithmetic kept for
    API parity (the device splits its own work)."""
    if t < 1:
        raise ValueError("chunk count must be at least 1")
    step = -(-nbytes // t)
    starts = np.minimum(np.arange(t, dtype=np.int64) * step, nbytes)
    stops = np.minimum(starts + step, nbytes)
    return [(int(a), int(b)) for a, b in zip(starts, stops)]


def and_masks_chunked(masks, t: int, pool=None) -> np.ndarray:
    """Bitwise AND of bitmasks (scan.py:55-78), computed on the GPU in one
    launch; ``t`` is validated like the reference but the device splits the
    work by itself."""
    masks = list(masks)
    if not masks:
        raise ValueError("no masks to merge")
    if t < 1:
        raise ValueError("chunk count must be at least 1")
    return kernels.and_masks(masks)


def mask_popcount(mask: np.ndarray) -> int:
    return kernels.mask_popcount(mask)


def mask_to_ids(mask: np.ndarray, n: int) -> np.ndarray:
    """Positions of set bits, ascending (scan.py:85-88)."""
    return kernels.mask_to_ids(mask, n)


class BatchResult:
    """Ids of a query batch: ``offsets`` int64[nq+1] into ``ids`` uint32."""

    __slots__ = ("offsets", "ids")

    def __init__(self, offsets: np.ndarray, ids: np.ndarray):
        self.offsets = offsets
        self.ids = ids

    def __len__(self) -> int:
        return int(self.offsets.size - 1)

    def counts(self) -> np.ndarray:
        return np.diff(self.offsets)

    def ids_of(self, q: int) -> np.ndarray:
        return self.ids[self.offsets[q]:self.offsets[q + 1]]

    def __getitem__(self, q: int) -> ResultSet:
        if not -len(self) <= q < len(self):
            raise IndexError(q)
        q %= len(self)
        return ResultSet(self.ids_of(q).astype(np.int64))

    def __iter__(self):
        for q in range(len(self)):
            yield self[q]


class _GpuScan:
    """Shared machinery: one device store + the reference search protocol."""

    name = "gpu"
    _path = "auto"          # one query: search() / search_with_stats()
    _batch_path = "auto"    # many: search_batch() / search_stream() -- the planner
    _layouts = _lib.LAYOUT_COLUMNAR

    def _open(self, values, device=None, va_bits=0):
        self.n, self.m = int(values.shape[0]), int(values.shape[1])
        self.store = DeviceStore(values, layouts=self._layouts, va_bits=va_bits, device=device)

    @property
    def size(self) -> int:
        return self.n

    def _check(self, query: RangeQuery):
        if query.m != self.m:
            raise ValueError(f"query has {query.m} dimensions, data has {self.m}")

    def search(self, query: RangeQuery) -> ResultSet:
        # the ids alone (search_with_stats adds the counters' readback)
        self._check(query)
        lo, hi = stack_queries([query], self.m)
        # int64 ids straight from the C ABI: the reference ResultSet dtype
        return ResultSet(self.store.ids64(lo, hi, self._path)[1])

    def _ids(self, queries, path=None):
        lo, hi = stack_queries(queries, self.m)
        offsets, ids = self.store.ids(lo, hi, path or self._path)
        return BatchResult(offsets, ids)

    def search_stream(self, batches, outs=None, info: dict | None = None) -> list:
        """Pipelined ids of a sequence of query batches (a serving loop /
        the reference harness's repetitions, bench.py:178-186): one
        BatchResult per batch; batch k's device->host copy runs under batch
        k+1's device pass (DeviceStore.ids_stream).  ``outs`` optionally
        gives one caller-owned (pinned) uint32 buffer per batch."""
        pairs, seen = [], {}
        for queries in batches:
            if id(queries) not in seen:   # a repeated batch object is stacked once
                qs = list(queries)
                for q in qs:
                    self._check(q)
                seen[id(queries)] = stack_queries(qs, self.m)
            pairs.append(seen[id(queries)])
        return [BatchResult(o, i) for o, i in self.store.ids_stream(pairs, self._batch_path, outs=outs, info=info)]

    def search_batch(self, queries) -> BatchResult:
        """Ids of every query of the batch, ascending per query."""
        queries = list(queries)
        for q in queries:
            self._check(q)
        return self._ids(queries, self._batch_path)

    def count(self, query: RangeQuery) -> int:
        self._check(query)
        return int(self.count_batch([query])[0])

    def count_batch(self, queries, path: str | None = None) -> np.ndarray:
        queries = list(queries)
        for q in queries:
            self._check(q)
        lo, hi = stack_queries(queries, self.m)
        return self.store.count(lo, hi, path or self._count_path)

    _count_path = "auto"

    def close(self) -> None:
        st = getattr(self, "store", None)
        if st is not None:
            st.close()


class SequentialScan(_GpuScan):
    """Row-wise scan over the whole dataset (scan.py:91-114), on the GPU."""

    _path = "rowwise"
    _count_path = "rowwise"
    _layouts = _lib.LAYOUT_ROWWISE

    def __init__(self, data: DataSet, mode: KernelMode = KernelMode.SCALAR, *, device: int | None = None):
        self.data = data
        self.mode = mode
        self.name = "sequential"
        self._open(data.values, device)

    def search_with_stats(self, query: RangeQuery) -> tuple[ResultSet, SearchStats]:
        self._check(query)
        lo, hi = stack_queries([query], self.m)
        _, ids, st = self.store.ids64_with_stats(
            lo, hi, self._path, MODE_BLOCKED if self.mode is KernelMode.VECTORIZED else MODE_SCALAR)
        return ResultSet(ids), SearchStats(objects_compared=self.n, early_breaks=int(st[0].early_breaks))


class HorizontalScan(_GpuScan):
    """Horizontal-partition scan (scan.py:117-164) on the GPU.

    The reference copies p random row partitions into blocks and merges
    per-partition ids with concatenate + sort.  Results do not depend on the
    layout (pinned by the reference's own tests, test_scan.py:84-89), so the
    GPU keeps one contiguous row-major store and emits ids already sorted;
    the layout is validated against the dataset exactly as the reference
    does.  Across GPUs the partitioning is contiguous row shards
    (parallel.ShardedScan).
    """

    _path = "rowwise"
    _count_path = "rowwise"
    _layouts = _lib.LAYOUT_ROWWISE

    def __init__(self, data: DataSet, layout: PartitionLayout, *, mode: KernelMode = KernelMode.SCALAR,
                 threads: int | None = None, device: int | None = None):
        if layout.n != data.n:
            raise ValueError(f"layout covers {layout.n} objects, dataset has {data.n}")
        self.m = data.m
        self.mode = mode
        self.layout = layout
        self.name = "horizontal"
        self._open(data.values, device)

    def search_with_stats(self, query: RangeQuery) -> tuple[ResultSet, SearchStats]:
        self._check(query)
        lo, hi = stack_queries([query], self.m)
        _, ids, st = self.store.ids64_with_stats(
            lo, hi, self._path, MODE_BLOCKED if self.mode is KernelMode.VECTORIZED else MODE_SCALAR)
        return ResultSet(ids), SearchStats(objects_compared=self.n, early_breaks=int(st[0].early_breaks))


class VerticalScan(_GpuScan):
    """Columnar scan (scan.py:167-214): unqueried dimensions are never read,
    a query with no queried dimension returns every id."""

    _path = "columnar"
    _count_path = "auto"
    _layouts = _lib.LAYOUT_COLUMNAR

    def __init__(self, source, *, threads: int | None = None, mode: KernelMode = KernelMode.VECTORIZED,
                 device: int | None = None):
        if isinstance(source, ColumnSet):
            values = source.to_matrix()
        elif isinstance(source, DataSet):
            values = source.values
        else:
            values = DataSet(source).values
        self.mode = mode
        self.t = threads if threads is not None else default_threads()
        self.name = "vertical"
        self._open(values, device)

    def search_with_stats(self, query: RangeQuery) -> tuple[ResultSet, SearchStats]:
        self._check(query)
        dims = query.queried_dims
        if dims.size == 0:   # scan.py:195-196
            return ResultSet(np.arange(self.n, dtype=np.int64)), SearchStats()
        res = self._ids([query])
        stats = SearchStats(objects_compared=int(dims.size) * self.n, columns_scanned=int(dims.size),
                            and_chunks=self.t)
        return res[0], stats


def sequential_scan(data: DataSet, query: RangeQuery, kernel: KernelMode = KernelMode.SCALAR) -> ResultSet:
    """One-shot sequential scan (scan.py:217-220)."""
    s = SequentialScan(data, kernel)
    try:
        return s.search(query)
    finally:
        s.close()


def horizontal_scan(data: DataSet, layout: PartitionLayout, query: RangeQuery,
                    kernel: KernelMode = KernelMode.SCALAR, threads: int | None = None) -> ResultSet:
    scanner = HorizontalScan(data, layout, mode=kernel, threads=threads)
    try:
        return scanner.search(query)
    finally:
        scanner.close()


def vertical_scan(cols, query: RangeQuery, workers: int) -> ResultSet:
    scanner = VerticalScan(cols, threads=workers)
    try:
        return scanner.search(query)
    finally:
        scanner.close()
