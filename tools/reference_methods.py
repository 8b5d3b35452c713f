"""CPU timings of the reference's own access methods ("CPU
side"), run on the GPU box's host cores:

    python tools/reference_methods.py > profiles/r01_reference_methods_box.json

The reference package comes from ``baseline/_ref`` (installed once in the
build container with ``pip install --no-index --no-build-isolation
--target baseline/_ref <copy of /root/reference/pkg>``; git-ignored, shipped
to the box by gpurun), else from a scratch build of /root/reference
(tests/golden/make_golden.py load_reference).  It is driven through its public API: build_method(name, data,
threads, mode) + search(query), median of 3 timed repetitions over a fixed
query subset after one warm-up query.  Data: C1 (1e6 x 3, seed 0, the
reference's gen_uniform) for the scans and the VA-file; the tree indexes are
built on the first 200 000 rows (Python R*-tree insertion costs ~75 us per row,
SURVEY.md 8(d) scale-downs), which is stated per entry.  These numbers come
from the host this runs on (os.cpu_count / physical cores / CPU model are
recorded).  A C2 leg (5e7 x 8, s = 1e-3, the bench workload) times the scans
on a few queries.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def _reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "mdrq")):
        sys.path.insert(0, ref)
        import mdrq
        assert mdrq.BACKEND == "compiled", mdrq.BACKEND
        return mdrq, "baseline/_ref (pip install of the reference package)"
    from make_golden import load_reference
    return load_reference(), "scratch build of /root/reference/pkg"


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _time(mdrq, name, mode, values, lo, hi, nq, threads):
    data = mdrq.DataSet(values)
    t0 = time.perf_counter()
    m = mdrq.build_method(name, data, threads=threads, mode=mdrq.KernelMode.parse(mode))
    build_s = time.perf_counter() - t0
    qs = [mdrq.RangeQuery(lo[i], hi[i]) for i in range(nq)]
    m.search(qs[0])
    reps = []
    for _ in range(3):
        t0 = time.perf_counter()
        for q in qs:
            m.search(q)
        reps.append(time.perf_counter() - t0)
    m.close()
    t = float(np.median(reps)) / nq
    return {"method": name, "mode": mode, "n": int(values.shape[0]), "m": int(values.shape[1]),
            "threads": threads, "queries": nq, "build_s": round(build_s, 2),
            "us_per_query": round(t * 1e6, 1), "tuples_per_s": values.shape[0] / t}


def bench_leg(threads: int | None = None) -> dict | None:
    """The bounded table bench.py prints beside its line (~20-30 s of host
    work): the reference's own scan, VA-file, kd-tree and R*-tree methods on
    C1 (the trees on a 1e5-row prefix), 10-20 queries each, from
    baseline/_ref.  None when the reference package is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mdrq")):
        return None
    import psutil
    from paper_1801_03644_b200 import workload
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import mdrq
    threads = threads or os.cpu_count() or 1
    values = workload.c1_data()
    lo, hi = workload.c1_queries()
    out = {"host_threads": threads, "physical_cores": psutil.cpu_count(logical=False), "cpu_model": _cpu_model(),
           "reference": f"baseline/_ref (backend {mdrq.BACKEND})",
           "data": "C1: 1e6 x 3 uniform seed 0, queries at 1 % selectivity; kd-tree / R*-tree on the first 1e5 rows",
           "methods": []}
    plan = [("sequential", "scalar", 1_000_000, 10), ("horizontal", "scalar", 1_000_000, 20),
            ("vertical", "scalar", 1_000_000, 10), ("vafile", "scalar", 1_000_000, 10),
            ("kdtree", "scalar", 100_000, 20), ("rstar", "scalar", 100_000, 20)]
    for name, mode, n, nq in plan:
        e = _time(mdrq, name, mode, values[:n], lo, hi, nq, threads)
        out["methods"].append({k: e[k] for k in ("method", "n", "queries", "build_s", "us_per_query")})
    return out


def main():
    import psutil
    from paper_1801_03644_b200 import workload
    mdrq, source = _reference()
    values = workload.c1_data()
    lo, hi = workload.c1_queries()
    threads = os.cpu_count() or 1
    out = {"host_threads": threads, "physical_cores": psutil.cpu_count(logical=False),
           "cpu_model": _cpu_model(), "reference": source,
           "data": "C1: 1e6 x 3 uniform seed 0, queries at 1 % selectivity", "methods": []}
    plan = [("sequential", "scalar", 1_000_000, 20), ("sequential", "vector", 1_000_000, 20),
            ("horizontal", "scalar", 1_000_000, 50), ("vertical", "scalar", 1_000_000, 50),
            ("vafile", "scalar", 1_000_000, 10), ("kdtree", "scalar", 200_000, 50),
            ("rstar", "scalar", 200_000, 50)]
    for name, mode, n, nq in plan:
        entry = _time(mdrq, name, mode, values[:n], lo, hi, nq, threads)
        entry["config"] = "C1" if n == values.shape[0] else f"C1 first {n} rows"
        out["methods"].append(entry)
        sys.stderr.write(json.dumps(entry) + "\n")
    # C2 (the bench workload): the scans on a few of its queries
    v2 = workload.c2_data()
    lo2, hi2 = workload.c2_queries(count=8, levels=(1e-3,))[1e-3]
    for name, mode, nq in [("sequential", "scalar", 2), ("horizontal", "scalar", 8), ("vertical", "scalar", 4)]:
        entry = _time(mdrq, name, mode, v2, lo2, hi2, nq, threads)
        entry["config"] = "C2 (5e7 x 8, s = 1e-3)"
        out["methods"].append(entry)
        sys.stderr.write(json.dumps(entry) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
