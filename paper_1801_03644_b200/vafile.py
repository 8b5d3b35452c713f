"""VA-file filter-and-refine on the GPU with a quantile grid.

Reference: /root/reference/pkg/src/mdrq/vafile.py -- a 2-bit equal-width
grid per dimension (VaGrid, vafile.py:25-64), a sparse code -> bucket
directory (vafile.py:106-147), candidate-cell enumeration
(vafile.py:154-199) and an exact ``scan_rows`` refine per candidate bucket
(vafile.py:204-219).

Here: per dimension 2^bits quantile cells (default
bits = 8) chosen from a strided device sample; every tuple is approximated
by one byte per dimension, stored as columnar byte planes in HBM.  A query
streams the byte planes of its queried dimensions, rejects tuples whose code
lies outside [code(lo), code(hi)], accepts tuples strictly inside, and
refines only tuples in an edge cell against the exact float32 columns.
``code(v) = #{boundaries <= v}`` makes the filter sound and the result
identical to the scan (parity is on id sets; the grid itself differs from
the reference's by design).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import DataSet, KernelMode, RangeQuery, ResultSet, SearchStats, stack_queries
from .scan import BatchResult
from .store import DEFAULT_VA_BITS, DeviceStore


class QuantileGrid:
    """Per-dimension sorted cell boundaries; the VaGrid API (vafile.py:25-64)
    for the quantile grid.  ``cell_index`` = number of boundaries <= value."""

    __slots__ = ("boundaries", "m", "bits")

    def __init__(self, boundaries: np.ndarray, bits: int):
        b = np.ascontiguousarray(boundaries, dtype=np.float32)
        if b.ndim != 2:
            raise ValueError("boundaries must have shape (m, 2^bits - 1)")
        self.boundaries = b
        self.m = b.shape[0]
        self.bits = bits

    @property
    def cells_per_dim(self) -> int:
        return 1 << self.bits

    def cell_index(self, value: float, dim: int) -> int:
        return int(np.searchsorted(self.boundaries[dim], np.float32(value), side="right"))

    def approximate(self, obj) -> np.ndarray:
        row = np.asarray(obj, dtype=np.float32)
        if row.shape != (self.m,):
            raise ValueError(f"object must have {self.m} dimensions")
        return np.array([self.cell_index(row[j], j) for j in range(self.m)], dtype=np.uint8)

    def approximate_all(self, values: np.ndarray) -> np.ndarray:
        vals = np.asarray(values, dtype=np.float32)
        out = np.empty(vals.shape, dtype=np.uint8)
        for j in range(self.m):
            out[:, j] = np.searchsorted(self.boundaries[j], vals[:, j], side="right")
        return out


class VaFile:
    """GPU VA-file over one device store (one instance per shard)."""

    name = "vafile"

    def __init__(self, store: DeviceStore, ids: np.ndarray | None, *, mode: KernelMode = KernelMode.SCALAR):
        self.store = store
        self.mode = mode
        self._ids = ids  # None = identity (ids 0..n-1)
        self.grid = QuantileGrid(store.va_boundaries(), store.va_bits)
        self.m = store.m

    @classmethod
    def build(cls, objects, ids, seed: int = 0, *, per_dim_bounds: np.ndarray | None = None,
              mode: KernelMode = KernelMode.SCALAR, bits: int = DEFAULT_VA_BITS,
              device: int | None = None) -> "VaFile":
        """Approximate every object and keep the byte planes in HBM
        (vafile.py:106-147).  ``seed`` / ``per_dim_bounds`` are accepted for
        factory-signature parity; the quantile grid does not use them."""
        objects = np.ascontiguousarray(objects, dtype=np.float32)
        if objects.ndim != 2:
            raise ValueError("objects must be a 2-d matrix")
        n = objects.shape[0]
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        if ids.shape != (n,):
            raise ValueError("ids must have one entry per object")
        identity = bool(n == 0 or (ids[0] == 0 and np.array_equal(ids, np.arange(n, dtype=np.int64))))
        store = DeviceStore(objects, layouts=_lib.LAYOUT_VAFILE, va_bits=bits, device=device)
        return cls(store, None if identity else ids, mode=mode)

    @classmethod
    def from_dataset(cls, data: DataSet, *, mode: KernelMode = KernelMode.SCALAR,
                     bits: int = DEFAULT_VA_BITS, device: int | None = None) -> "VaFile":
        store = DeviceStore(data.values, layouts=_lib.LAYOUT_VAFILE, va_bits=bits, device=device)
        return cls(store, None, mode=mode)

    @property
    def size(self) -> int:
        return self.store.n

    def _map(self, local: np.ndarray) -> np.ndarray:
        if self._ids is None:
            return local if local.dtype == np.int64 else local.astype(np.int64)
        return np.sort(self._ids[local.astype(np.int64)])

    def search(self, query: RangeQuery) -> ResultSet:
        # the ids alone (search_with_stats adds the counters' readback)
        if query.m != self.m:
            raise ValueError(f"query has {query.m} dimensions, grid has {self.m}")
        lo, hi = stack_queries([query], self.m)
        offs, ids = self.store.ids64(lo, hi, "vafile")
        return ResultSet(self._map(ids))

    def search_with_stats(self, query: RangeQuery) -> tuple[ResultSet, SearchStats]:
        if query.m != self.m:
            raise ValueError(f"query has {query.m} dimensions, grid has {self.m}")
        lo, hi = stack_queries([query], self.m)
        offs, ids, st = self.store.ids64_with_stats(lo, hi, "vafile")
        st = st[0]
        stats = SearchStats(objects_compared=int(st.objects_compared), nodes_visited=int(st.nodes_visited),
                            columns_scanned=int(st.columns_scanned))
        return ResultSet(self._map(ids)), stats

    def search_batch(self, queries) -> BatchResult:
        queries = list(queries)
        for q in queries:
            if q.m != self.m:
                raise ValueError(f"query has {q.m} dimensions, grid has {self.m}")
        lo, hi = stack_queries(queries, self.m)
        # the planner: a batch whose queries' dims sum to >= 10x the union's
        # (10 full-match queries) goes through the bit-sliced multi-query
        # pass (<= 1024 queries per pass over the code planes)
        offs, ids = self.store.ids(lo, hi, "auto")
        if self._ids is not None:
            parts = [self._map(ids[offs[q]:offs[q + 1]]) for q in range(len(queries))]
            ids = np.concatenate(parts) if parts else np.empty(0, np.int64)
        return BatchResult(offs, ids)

    def count(self, query: RangeQuery) -> int:
        return int(self.count_batch([query])[0])

    def count_batch(self, queries) -> np.ndarray:
        queries = list(queries)
        for q in queries:
            if q.m != self.m:
                raise ValueError(f"query has {q.m} dimensions, grid has {self.m}")
        lo, hi = stack_queries(queries, self.m)
        return self.store.count(lo, hi, "auto")

    def search_stream(self, batches, outs=None, info: dict | None = None) -> list:
        """Pipelined ids of a sequence of query batches (see
        _GpuScan.search_stream)."""
        pairs, seen = [], {}
        for queries in batches:
            if id(queries) not in seen:   # a repeated batch object is stacked once
                qs = list(queries)
                for q in qs:
                    if q.m != self.m:
                        raise ValueError(f"query has {q.m} dimensions, grid has {self.m}")
                seen[id(queries)] = stack_queries(qs, self.m)
            pairs.append(seen[id(queries)])
        res = self.store.ids_stream(pairs, "auto", outs=outs, info=info)
        if self._ids is not None:
            out = []
            for offs, ids in res:
                parts = [self._map(ids[offs[q]:offs[q + 1]]) for q in range(offs.size - 1)]
                out.append(BatchResult(offs, np.concatenate(parts) if parts else np.empty(0, np.int64)))
            return out
        return [BatchResult(o, i) for o, i in res]

    def close(self) -> None:
        self.store.close()
