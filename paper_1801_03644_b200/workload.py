"""Synthetic data and query generators for the hot path's configurations.

``gen_uniform`` is the reference's own generator, bit for bit
(/root/reference/pkg/src/mdrq/workload.py:59-65:
``np.random.default_rng(seed).random((n, m), dtype=np.float32)``);
``gen_query_from_pair`` / ``pair_query_batch`` restate workload.py:113-126;
``write_queries`` / ``read_queries`` the JSONL query format
(workload.py:343-366).

The BASELINE.json configurations:

* C1: n=1e6, m=3 uniform (seed 0); 1000 full-match queries, width
  0.01**(1/3), lower bound U[0, 1-w) from default_rng(1);
* C2: n=5e7, m=8 uniform (seed 0); 1000 queries per selectivity level
  s in (1e-5, 1e-4, 1e-3, 1e-2, 1e-1), width s**(1/8), one default_rng(1)
  drawn level after level;
* C5: n=5e8, m=10 uniform (seed 0); 10000 queries, width 0.001**0.1.

Uniform data can be generated shard by shard (``uniform_rows``) with the
PCG64 stream advanced to the shard's first value -- identical to slicing
the one-shot array (tests/test_workload.py).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .core import DataSet, RangeQuery


@dataclass(frozen=True)
class GeneratorSpec:
    """workload.py:38-56 (the clustered kind is out of scope here)."""

    kind: str
    n: int
    m: int
    cluster_count: int = 1
    cluster_extent: float = 0.1
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("uniform", "clustered"):
            raise ValueError(f"unknown generator kind {self.kind!r}")
        if self.n < 0 or self.m < 1:
            raise ValueError("need n >= 0 and m >= 1")


def gen_uniform(spec: GeneratorSpec) -> DataSet:
    """n*m independent float32 draws from [0, 1), seeded (workload.py:59-65)."""
    if spec.kind != "uniform":
        raise ValueError("spec.kind must be 'uniform'")
    rng = np.random.default_rng(spec.seed)
    return DataSet(rng.random((spec.n, spec.m), dtype=np.float32))


def gen_dataset(spec: GeneratorSpec) -> DataSet:
    if spec.kind != "uniform":
        raise ValueError("only the uniform generator is part of the GPU hot path's workloads")
    return gen_uniform(spec)


def uniform_rows(seed: int, m: int, start: int, stop: int) -> np.ndarray:
    """Rows [start, stop) of ``default_rng(seed).random((n, m), float32)``
    without generating the prefix: PCG64 emits 64-bit words and float32
    draws consume 32-bit halves, so the stream is advanced by
    (start*m)//2 words and an odd half is drawn and dropped."""
    if stop < start:
        raise ValueError("stop < start")
    bg = np.random.PCG64(seed)
    first = start * m
    bg.advance(first // 2)
    rng = np.random.Generator(bg)
    if first % 2:
        rng.random(1, dtype=np.float32)
    return rng.random((stop - start, m), dtype=np.float32)


def _generator(seed) -> np.random.Generator:
    return seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)


def gen_query_from_pair(data: DataSet, seed) -> RangeQuery:
    """The bounding box of two distinct random objects (workload.py:113-120):
    one ``choice(n, 2, replace=False)`` draw per query, so a shared generator
    yields the reference's query sequence."""
    if data.n < 2:
        raise ValueError("pair query generation needs at least 2 objects")
    pair = data.values[_generator(seed).choice(data.n, size=2, replace=False)]
    return RangeQuery(pair.min(axis=0), pair.max(axis=0))


def pair_query_batch(data: DataSet, count: int, seed) -> list[RangeQuery]:
    """``count`` pair queries from one generator (workload.py:123-126)."""
    rng = _generator(seed)
    return [gen_query_from_pair(data, rng) for _ in range(count)]


# -- BASELINE configurations --------------------------------------------------

C1 = dict(n=1_000_000, m=3, queries=1000, selectivity=0.01)
C2 = dict(n=50_000_000, m=8, queries=1000, levels=(1e-5, 1e-4, 1e-3, 1e-2, 1e-1))
C5 = dict(n=500_000_000, m=10, queries=10_000, selectivity=1e-3)


def box_queries(rng: np.random.Generator, count: int, m: int, selectivity: float):
    """Full-match boxes of per-dimension width s**(1/m) with lower bounds
    U[0, 1-w) (float64 draws, cast to float32 like RangeQuery, core.py:119-120)."""
    w = selectivity ** (1.0 / m)
    lo = rng.uniform(0.0, 1.0 - w, (count, m))
    hi = lo + w
    return lo.astype(np.float32), hi.astype(np.float32)


def c1_data() -> np.ndarray:
    return np.random.default_rng(0).random((C1["n"], C1["m"]), dtype=np.float32)


def c1_queries(count: int = C1["queries"]):
    return box_queries(np.random.default_rng(1), count, C1["m"], C1["selectivity"])


def c2_data(n: int = C2["n"], start: int = 0, stop: int | None = None) -> np.ndarray:
    stop = n if stop is None else stop
    if start == 0 and stop == n:
        return np.random.default_rng(0).random((n, C2["m"]), dtype=np.float32)
    return uniform_rows(0, C2["m"], start, stop)


def c2_queries(count: int = C2["queries"], levels=C2["levels"]):
    """{selectivity: (lo, hi)} drawn level after level from default_rng(1)."""
    rng = np.random.default_rng(1)
    return {s: box_queries(rng, count, C2["m"], s) for s in levels}


def _uniform_chunk_fn(seed: int, m: int):
    return _UniformChunk(seed, m)


class _UniformChunk:
    """Picklable chunk generator of default_rng(seed).random((n, m), f32)."""

    def __init__(self, seed: int, m: int):
        self.seed, self.m = seed, m

    def __call__(self, c: int, rows: int) -> np.ndarray:
        return uniform_rows(self.seed, self.m, c * CHUNK_ROWS, c * CHUNK_ROWS + rows)


def c5_data(start: int = 0, stop: int | None = None, n: int = C5["n"], workers: int | None = None) -> np.ndarray:
    """Rows [start, stop) of C5 (= default_rng(0).random((5e8, 10), float32)),
    generated chunk-parallel with the PCG64 stream advanced per chunk."""
    stop = n if stop is None else stop
    return _chunked(_uniform_chunk_fn(0, C5["m"]), C5["m"], start, stop, n, workers)


def c5_queries(count: int = C5["queries"]):
    return box_queries(np.random.default_rng(1), count, C5["m"], C5["selectivity"])


C3 = dict(n=100_000_000, m=16, queries=2000, centres=20, sigma=0.03, zipf=1.1, sel=(1e-3, 5e-2))
C4 = dict(n=10_000_000, m=19, queries=5000)
CHUNK_ROWS = 1 << 20  # generation chunk of the clustered / mixed configs


def _chunks(start: int, stop: int):
    """(chunk index, row range within the chunk) covering rows [start, stop)."""
    c = start // CHUNK_ROWS
    while c * CHUNK_ROWS < stop:
        a = max(start, c * CHUNK_ROWS) - c * CHUNK_ROWS
        b = min(stop, (c + 1) * CHUNK_ROWS) - c * CHUNK_ROWS
        yield c, a, b
        c += 1


def c3_model():
    """Gaussian-mixture model of C3: 20 centres U[0,1)^16 (default_rng(3)),
    Zipf(1.1) weights, per-dimension sigma 0.03."""
    centres = np.random.default_rng(3).random((C3["centres"], C3["m"]))
    w = 1.0 / np.arange(1, C3["centres"] + 1) ** C3["zipf"]
    return centres, w / w.sum()


def c3_chunk(c: int, rows: int | None = None) -> np.ndarray:
    """Chunk c (CHUNK_ROWS rows) of C3: default_rng([3, c]) draws the cluster
    of every row (choice) then the N(0, sigma) noise; values are clipped to
    [0, nextafter(1, 0)] in float32."""
    rows = CHUNK_ROWS if rows is None else rows
    centres, p = c3_model()
    rng = np.random.default_rng([3, c])
    assign = rng.choice(C3["centres"], size=rows, p=p)
    noise = rng.normal(0.0, C3["sigma"], (rows, C3["m"]))
    v = (centres[assign] + noise).astype(np.float32)
    np.clip(v, np.float32(0.0), np.nextafter(np.float32(1.0), np.float32(0.0)), out=v)
    return v


def _chunked(chunk_fn, m: int, start: int, stop: int, n: int, workers: int | None) -> np.ndarray:
    """Rows [start, stop) of a chunk-generated table; chunks are independent
    (seeded by their index), so they are generated in parallel worker
    processes writing straight into shared memory."""
    import os
    out_shape = (stop - start, m)
    jobs = list(_chunks(start, stop))
    workers = workers or min(len(jobs), os.cpu_count() or 1)
    if workers <= 1 or len(jobs) <= 1:
        out = np.empty(out_shape, np.float32)
        o = 0
        for c, a, b in jobs:
            out[o:o + b - a] = chunk_fn(c, min(CHUNK_ROWS, n - c * CHUNK_ROWS))[a:b]
            o += b - a
        return out
    import multiprocessing as mp
    from multiprocessing import shared_memory
    import weakref
    shm = shared_memory.SharedMemory(create=True, size=max(1, out_shape[0] * m * 4))
    try:
        offs = []
        o = 0
        for c, a, b in jobs:
            offs.append(o)
            o += b - a
        # spawn, not fork: the caller may already run CUDA / torch threads
        ctx = mp.get_context("spawn")
        with ctx.Pool(workers) as pool:
            pool.starmap(_fill_chunk, [(chunk_fn, shm.name, out_shape, off, c, a, b, n, m)
                                       for off, (c, a, b) in zip(offs, jobs)])
    finally:
        shm.unlink()   # the mapping stays valid until the array below is freed
    out = np.ndarray(out_shape, np.float32, buffer=shm.buf)
    weakref.finalize(out, shm.close)
    return out


def _fill_chunk(chunk_fn, name, shape, off, c, a, b, n, m):
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(name=name)
    try:
        dst = np.ndarray(shape, np.float32, buffer=shm.buf)
        dst[off:off + b - a] = chunk_fn(c, min(CHUNK_ROWS, n - c * CHUNK_ROWS))[a:b]
    finally:
        shm.close()


def c3_data(start: int = 0, stop: int | None = None, n: int = C3["n"], workers: int | None = None) -> np.ndarray:
    stop = n if stop is None else stop
    return _chunked(c3_chunk, C3["m"], start, stop, n, workers)


def _tune_halfwidth(sample: np.ndarray, centre: np.ndarray, dims: np.ndarray, target: float) -> float:
    """Bisection on the common half-width so the box around `centre` on
    `dims` selects ~target of `sample` (mirrors the reference's
    selectivity-bucket tuning, bench.py:215-252)."""
    cols = sample[:, dims]
    c = centre[dims]
    lo_h, hi_h = 0.0, 1.0
    for _ in range(22):
        h = 0.5 * (lo_h + hi_h)
        sel = np.count_nonzero((np.abs(cols - c) <= h).all(axis=1)) / sample.shape[0]
        if sel < target:
            lo_h = h
        else:
            hi_h = h
    return hi_h


def c3_queries(count: int = C3["queries"], sample_rows: int = 1 << 18):
    """C3 partial-match queries: k ~ U{2..8} of the 16 dims, centred on a
    random tuple of chunk 0, half-width tuned by bisection on a sample of
    chunk 0 for a log-uniform target selectivity in [1e-3, 5e-2]."""
    rng = np.random.default_rng(4)
    chunk0 = c3_chunk(0)
    sample = chunk0[:sample_rows]
    m = C3["m"]
    lo = np.full((count, m), -np.inf, np.float32)
    hi = np.full((count, m), np.inf, np.float32)
    a, b = np.log(C3["sel"][0]), np.log(C3["sel"][1])
    for q in range(count):
        k = int(rng.integers(2, 9))
        dims = np.sort(rng.choice(m, size=k, replace=False))
        centre = chunk0[int(rng.integers(0, CHUNK_ROWS))]
        target = float(np.exp(rng.uniform(a, b)))
        h = _tune_halfwidth(sample, centre, dims, target)
        lo[q, dims] = (centre[dims] - h).astype(np.float32)
        hi[q, dims] = (centre[dims] + h).astype(np.float32)
    return lo, hi


_C4_CARDS = (2, 3, 5, 10, 25, 50)
_C4_NORMAL = ((45.0, 15.0), (70.0, 15.0), (120.0, 20.0), (25.0, 5.0), (60.0, 10.0))


def _zipf_p(k: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, k + 1) ** s
    return w / w.sum()


def c4_chunk(c: int, rows: int | None = None) -> np.ndarray:
    """Chunk c of C4 (genomics-shaped, 19 float32 columns, default_rng([4, c])):
    d0 chromosome 1..25 Zipf(1.0); d1 position U{0..2.5e8-1} (float32, exact
    only to multiples of 16 above 2^24); d2-d7 categoricals of cardinality
    2, 3, 5, 10, 25, 50 with Zipf(1.2) frequencies; d8-d12 normal values
    rounded to integers and clipped to [0, 250]; d13-d18 U[0, 1)."""
    rows = CHUNK_ROWS if rows is None else rows
    rng = np.random.default_rng([4, c])
    v = np.empty((rows, 19), np.float32)
    v[:, 0] = rng.choice(np.arange(1, 26), size=rows, p=_zipf_p(25, 1.0))
    v[:, 1] = rng.integers(0, 250_000_000, size=rows).astype(np.float32)
    for j, card in enumerate(_C4_CARDS):
        v[:, 2 + j] = rng.choice(card, size=rows, p=_zipf_p(card, 1.2))
    for j, (mu, sd) in enumerate(_C4_NORMAL):
        v[:, 8 + j] = np.clip(np.rint(rng.normal(mu, sd, rows)), 0, 250)
    v[:, 13:] = rng.random((rows, 6), dtype=np.float32)
    return v


def c4_data(start: int = 0, stop: int | None = None, n: int = C4["n"], workers: int | None = None) -> np.ndarray:
    stop = n if stop is None else stop
    return _chunked(c4_chunk, 19, start, stop, n, workers)


def c4_queries(count: int = C4["queries"]):
    """C4 partial-match queries on 3-5 dims around a random tuple of chunk 0:
    equality (lo == hi) on categorical / integer dims (d0, d2-d12), an
    interval of log-uniform relative width on d1 and d13-d18 -- selectivities
    spread over ~1e-7..1e-2 (exact values from the oracle)."""
    rng = np.random.default_rng(5)
    chunk0 = c4_chunk(0)
    lo = np.full((count, 19), -np.inf, np.float32)
    hi = np.full((count, 19), np.inf, np.float32)
    for q in range(count):
        k = int(rng.integers(3, 6))
        dims = np.sort(rng.choice(19, size=k, replace=False))
        row = chunk0[int(rng.integers(0, CHUNK_ROWS))]
        for j in dims:
            v = row[j]
            if j == 1:
                w = np.float32(2.5e8 * np.exp(rng.uniform(np.log(1e-4), np.log(0.3))))
                lo[q, j], hi[q, j] = v - w / 2, v + w / 2
            elif j >= 13:
                w = np.float32(np.exp(rng.uniform(np.log(1e-3), np.log(0.5))))
                lo[q, j], hi[q, j] = v - w / 2, v + w / 2
            else:
                lo[q, j] = hi[q, j] = v
    return lo, hi


def queries_from_arrays(lo: np.ndarray, hi: np.ndarray) -> list[RangeQuery]:
    return [RangeQuery(lo[i], hi[i]) for i in range(lo.shape[0])]


# -- query batch serialisation (JSON lines, workload.py:343-366) ----------------

def _json_bound(v, sentinel):
    return None if v == sentinel else float(v)


def write_queries(queries, path) -> None:
    """JSON lines ``{"lower": [...], "upper": [...]}``; null stands for the
    -inf / +inf sentinel of an unqueried bound."""
    lines = [json.dumps({"lower": [_json_bound(v, -np.inf) for v in q.lower],
                         "upper": [_json_bound(v, np.inf) for v in q.upper]})
             for q in queries]
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(line + "\n" for line in lines)


def read_queries(path) -> list[RangeQuery]:
    """Inverse of ``write_queries``; blank lines are skipped, a malformed
    record raises ValueError naming ``path:line`` (workload.py:355-366)."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, text in enumerate(fh, 1):
            if not text.strip():
                continue
            try:
                rec = json.loads(text)
                lower = [-np.inf if v is None else v for v in rec["lower"]]
                upper = [np.inf if v is None else v for v in rec["upper"]]
            except (json.JSONDecodeError, KeyError, TypeError) as exc:
                raise ValueError(f"{path}:{lineno}: bad query record: {exc}") from None
            out.append(RangeQuery(lower, upper))
    return out
