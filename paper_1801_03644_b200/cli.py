"""Command line for the GPU methods.

    python -m paper_1801_03644_b200 verify --n 100000 --dims 5 --count 200
    python -m paper_1801_03644_b200 bench  --n 1000000 --dims 3 --queries 1000 --out r.csv

``verify`` restates the reference's oracle-equivalence audit
(cli.py:210-246): every GPU method's id set for every query must equal the
ground truth computed ON THE CPU -- the reference's own
``SequentialScan(KernelMode.SCALAR)`` (cli.py:222) when the reference package
``mdrq`` is importable (``--reference`` path, default baseline/_ref), else a
numpy containment test (the reference suite's independent oracle,
pkg/tests/test_scan.py:22-28); exit code 2 on a mismatch.
``bench`` restates run_benchmark (bench.py:146-212): build, one untimed
warm-up batch, the median of ``--repetitions`` timed batches (each batch one
``search_batch`` call over all queries), selectivity from the exact counts,
and a CSV report with the reference's columns (bench.py:34-38).
"""

from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time

import numpy as np

REPORT_COLUMNS = (
    "method", "n", "m", "threads", "partitions", "kernel", "clusters",
    "avg_selectivity", "queries", "seconds", "qps",
    "objects_compared", "nodes_visited",
)


def _data_and_queries(args):
    from .core import read_dataset
    from .workload import GeneratorSpec, gen_dataset, pair_query_batch, read_queries
    if args.data:
        data = read_dataset(args.data)
    else:
        data = gen_dataset(GeneratorSpec("uniform", args.n, args.dims, seed=args.seed))
    if args.queries_file:
        queries = read_queries(args.queries_file)
    else:
        queries = pair_query_batch(data, args.count, args.seed + 1)
    return data, queries


def _methods(spec: str):
    from .methods import METHOD_NAMES
    names = [s.strip() for s in spec.split(",") if s.strip()]
    for n in names:
        if n not in METHOD_NAMES:
            raise SystemExit(f"unknown method {n!r} (choose from {', '.join(METHOD_NAMES)})")
    return names


def _reference_module(path):
    """The reference package ``mdrq`` (compiled backend), or None."""
    import importlib
    if path and os.path.isdir(os.path.join(path, "mdrq")) and path not in sys.path:
        sys.path.insert(0, path)
    try:
        return importlib.import_module("mdrq")
    except ImportError:
        return None


def ground_truth(data, queries, reference_path=None):
    """CPU ground truth per query -> (list of int64 id arrays, source)."""
    ref = _reference_module(reference_path)
    if ref is not None and hasattr(ref, "SequentialScan"):
        scan = ref.SequentialScan(ref.DataSet(data.values), ref.KernelMode.SCALAR)
        try:
            exp = [scan.search(ref.RangeQuery(q.lower, q.upper)).ids for q in queries]
        finally:
            getattr(scan, "close", lambda: None)()
        return exp, f"reference SequentialScan(SCALAR) (mdrq backend {getattr(ref, 'BACKEND', '?')})"
    v = data.values
    exp = []
    for q in queries:
        ok = np.ones(v.shape[0], dtype=bool)
        for j in range(v.shape[1]):
            ok &= (v[:, j] >= q.lower[j]) & (v[:, j] <= q.upper[j])
        exp.append(np.flatnonzero(ok).astype(np.int64))
    return exp, "numpy containment on the CPU (pkg/tests/test_scan.py:22-28)"


def cmd_verify(args) -> int:
    from .core import KernelMode
    from .methods import build_method
    data, queries = _data_and_queries(args)
    ref_path = args.reference if args.reference is not None else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    expected, source = ground_truth(data, queries, ref_path)
    print(f"ground truth: {source}, {len(queries)} queries")
    failures = 0
    for name in _methods(args.method):
        method = build_method(name, data, threads=args.threads, mode=KernelMode.parse(args.kernel), seed=args.seed)
        bad = 0
        try:
            got = method.search_batch(queries)
            for qi in range(len(queries)):
                g, e = got.ids_of(qi).astype(np.int64), expected[qi]
                if not np.array_equal(g, e):
                    missing = np.setdiff1d(e, g)
                    extra = np.setdiff1d(g, e)
                    print(f"FAIL ({name}, query {qi}, missing={missing[:10].tolist()} extra={extra[:10].tolist()})")
                    bad += 1
        finally:
            method.close()
        failures += bad
        print(f"{name}: {'ok' if bad == 0 else 'MISMATCH'} ({len(queries)} queries)")
    if failures:
        print(f"verification failed: {failures} mismatching result sets")
        return 2
    print("verification passed: all methods match the CPU ground truth")
    return 0


def cmd_bench(args) -> int:
    from .core import KernelMode
    from .methods import build_method
    data, queries = _data_and_queries(args)
    rows = []
    for name in _methods(args.method):
        t0 = time.perf_counter()
        method = build_method(name, data, threads=args.threads, mode=KernelMode.parse(args.kernel), seed=args.seed)
        build_s = time.perf_counter() - t0
        try:
            warm = method.search_batch(queries)          # untimed warm-up
            total = int(warm.offsets[-1])
            times = []
            for _ in range(args.repetitions):
                t0 = time.perf_counter()
                res = method.search_batch(queries)
                times.append(time.perf_counter() - t0)
                if int(res.offsets[-1]) != total:
                    raise RuntimeError("timed run returned a different result total")
        finally:
            method.close()
        seconds = statistics.median(times)
        sel = float(np.mean(np.diff(warm.offsets) / max(data.n, 1))) if len(queries) else 0.0
        row = {"method": name, "n": data.n, "m": data.m, "threads": args.threads or 1,
               "partitions": args.threads or 1, "kernel": args.kernel, "clusters": 0,
               "avg_selectivity": sel, "queries": len(queries), "seconds": seconds,
               "qps": len(queries) / seconds if seconds > 0 else float("inf"),
               "objects_compared": data.n * len(queries), "nodes_visited": 0}
        rows.append(row)
        print(f"{name}: n={data.n} m={data.m} sel={sel:.4%} qps={row['qps']:.1f} build={build_s:.2f}s")
    if args.out:
        with open(args.out, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(REPORT_COLUMNS)
            for r in rows:
                w.writerow([f"{r[c]:.6g}" if isinstance(r[c], float) else str(r[c]) for c in REPORT_COLUMNS])
        print(f"wrote CSV report to {args.out}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1801_03644_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("verify", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--method", default="sequential,vertical,vafile" if name == "verify" else "vafile")
        p.add_argument("--n", type=int, default=100_000)
        p.add_argument("--dims", type=int, default=5)
        p.add_argument("--count", "--queries", dest="count", type=int, default=200)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--threads", type=int, default=None)
        p.add_argument("--kernel", default="scalar")
        p.add_argument("--data", default=None, help="dataset file (reference binary format)")
        p.add_argument("--queries-file", default=None, help="JSONL query batch")
        if name == "verify":
            p.add_argument("--reference", default=None,
                           help="directory holding the reference package mdrq (default baseline/_ref)")
        if name == "bench":
            p.add_argument("--repetitions", type=int, default=3)
            p.add_argument("--out", default=None)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.cmd == "verify":
        return cmd_verify(args)
    return cmd_bench(args)


if __name__ == "__main__":
    sys.exit(main())
