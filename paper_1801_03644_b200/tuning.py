"""GPU count service for workload tuning.

The reference tunes query workloads with exact counts on the CPU:
``selectivity_oracle`` (core.py:275-292, one scan per query) and
``collect_selectivity_buckets`` (bench.py:215-252: draw pair queries,
prefilter by a subsample estimate, assign by the exact oracle).  Here the
exact counts come from one multi-query pass over the device store, so the
candidates are counted on the FULL table in batches of thousands and no
subsample estimate is needed; the contract -- every returned query's exact
selectivity lies in its bucket -- is the reference's.
"""

from __future__ import annotations

import numpy as np

from .core import NEG_INF, POS_INF, DataSet, RangeQuery
from .store import DeviceStore
from . import _lib


def _pair_bounds(values: np.ndarray, rng: np.random.Generator, count: int):
    """Pair queries exactly as workload.gen_query_from_pair draws them
    (workload.py:113-120): two distinct random objects, per-dim min/max."""
    n = values.shape[0]
    lo = np.empty((count, values.shape[1]), np.float32)
    hi = np.empty_like(lo)
    for i in range(count):
        a, b = rng.choice(n, size=2, replace=False)
        lo[i] = np.minimum(values[a], values[b])
        hi[i] = np.maximum(values[a], values[b])
    return lo, hi


def collect_selectivity_buckets(data: DataSet, buckets, per_bucket: int, seed, *,
                                batch: int = 2048, max_draws: int = 300_000,
                                store: DeviceStore | None = None):
    """Pair-generated queries binned by exact selectivity (bench.py:215-252).

    Returns one list of RangeQuery per bucket (may fall short of per_bucket
    if the distribution is too thin within max_draws)."""
    if data.n < 2:
        raise ValueError("pair query generation needs at least 2 objects")
    rng = np.random.default_rng(seed)
    own = store is None
    if own:
        store = DeviceStore(data.values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8)
    out = [[] for _ in buckets]
    try:
        drawn = 0
        while drawn < max_draws and not all(len(qs) >= per_bucket for qs in out):
            k = min(batch, max_draws - drawn)
            lo, hi = _pair_bounds(data.values, rng, k)
            drawn += k
            sel = store.count(lo, hi) / data.n
            for i in range(k):
                for b, (blo, bhi) in enumerate(buckets):
                    if len(out[b]) < per_bucket and blo <= sel[i] <= bhi:
                        out[b].append(RangeQuery(lo[i], hi[i]))
                        break
    finally:
        if own:
            store.close()
    return out


def selectivities(data_or_store, queries) -> np.ndarray:
    """Exact joint selectivity of every query, one device pass."""
    from .core import stack_queries
    st = data_or_store if isinstance(data_or_store, DeviceStore) else DeviceStore(data_or_store.values)
    try:
        lo, hi = stack_queries(list(queries), st.m)
        return st.count(lo, hi) / max(st.n, 1)
    finally:
        if st is not data_or_store:
            st.close()


def tune_halfwidth(store: DeviceStore, centre: np.ndarray, dims: np.ndarray, target: float,
                   steps: int = 22, probes: int = 32) -> float:
    """Common half-width of a box around `centre` on `dims` whose exact
    selectivity on the whole table is closest to `target`: a batched
    bisection, `probes` widths counted per device pass (the GPU counterpart
    of workload._tune_halfwidth's sample bisection)."""
    m = store.m
    lo_h, hi_h = 0.0, 1.0
    best = 1.0
    for _ in range(max(1, steps // 5)):
        hs = np.linspace(lo_h, hi_h, probes + 2)[1:-1]
        lo = np.full((probes, m), NEG_INF, np.float32)
        hi = np.full((probes, m), POS_INF, np.float32)
        for i, h in enumerate(hs):
            lo[i, dims] = centre[dims] - h
            hi[i, dims] = centre[dims] + h
        sel = store.count(lo, hi) / store.n
        j = int(np.searchsorted(sel, target))
        lo_h = hs[j - 1] if j > 0 else lo_h
        hi_h = hs[j] if j < probes else hi_h
        best = hi_h
    return float(best)
