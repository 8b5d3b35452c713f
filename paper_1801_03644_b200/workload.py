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


def gen_query_from_pair(data: DataSet, seed) -> RangeQuery:
    """Complete-match query from two random objects (workload.py:113-120)."""
    if data.n < 2:
        raise ValueError("pair query generation needs at least 2 objects")
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    i, j = rng.choice(data.n, size=2, replace=False)
    a = data.values[i]
    b = data.values[j]
    return RangeQuery(np.minimum(a, b), np.maximum(a, b))


def pair_query_batch(data: DataSet, count: int, seed) -> list[RangeQuery]:
    """workload.py:123-126."""
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
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


def c5_data(start: int = 0, stop: int | None = None, n: int = C5["n"]) -> np.ndarray:
    stop = n if stop is None else stop
    return uniform_rows(0, C5["m"], start, stop)


def c5_queries(count: int = C5["queries"]):
    return box_queries(np.random.default_rng(1), count, C5["m"], C5["selectivity"])


def queries_from_arrays(lo: np.ndarray, hi: np.ndarray) -> list[RangeQuery]:
    return [RangeQuery(lo[i], hi[i]) for i in range(lo.shape[0])]


# -- query batch serialisation (JSON lines, workload.py:343-366) ----------------

def write_queries(queries, path) -> None:
    """One JSON object per line; nulls encode the infinity sentinels."""
    with open(path, "w", encoding="utf-8") as fh:
        for q in queries:
            lower = [None if v == -np.inf else float(v) for v in q.lower]
            upper = [None if v == np.inf else float(v) for v in q.upper]
            fh.write(json.dumps({"lower": lower, "upper": upper}) + "\n")


def read_queries(path) -> list[RangeQuery]:
    queries = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line:
                continue
            try:
                obj = json.loads(line)
                lower = [(-np.inf if v is None else v) for v in obj["lower"]]
                upper = [(np.inf if v is None else v) for v in obj["upper"]]
            except (json.JSONDecodeError, KeyError, TypeError) as exc:
                raise ValueError(f"{path}:{lineno}: bad query record: {exc}") from None
            queries.append(RangeQuery(lower, upper))
    return queries
