"""CPU timings of the reference's own access methods ("CPU
side"), run in the build container where /root/reference exists:

    python tools/reference_methods.py > profiles/r01_reference_methods.json

The reference package is built in a scratch copy (tests/golden/make_golden.py
load_reference) and driven through its public API: build_method(name, data,
threads, mode) + search(query), median of 3 timed repetitions over a fixed
query subset after one warm-up query.  Data: C1 (1e6 x 3, seed 0, the
reference's gen_uniform) for the scans and the VA-file; the tree indexes are
built on the first 200 000 rows (Python R*-tree insertion costs ~75 us per row,
SURVEY.md 8(d) scale-downs), which is stated per entry.  These numbers come
from this container's CPU, not the GPU box: bench.py's cpu_baseline is the
same-box baseline; this table is the method comparison the paper makes.
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


def main():
    from make_golden import load_reference
    from paper_1801_03644_b200 import workload
    mdrq = load_reference()
    values = workload.c1_data()
    lo, hi = workload.c1_queries()
    threads = os.cpu_count() or 1
    out = {"host_threads": threads, "data": "C1: 1e6 x 3 uniform seed 0, queries at 1 % selectivity",
           "methods": []}
    plan = [("sequential", "scalar", 1_000_000, 20), ("sequential", "vector", 1_000_000, 20),
            ("horizontal", "scalar", 1_000_000, 50), ("vertical", "scalar", 1_000_000, 50),
            ("vafile", "scalar", 1_000_000, 10), ("kdtree", "scalar", 200_000, 50),
            ("rstar", "scalar", 200_000, 50)]
    for name, mode, n, nq in plan:
        data = mdrq.DataSet(values[:n])
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
        entry = {"method": name, "mode": mode, "n": n, "queries": nq, "build_s": round(build_s, 2),
                 "us_per_query": round(t * 1e6, 1), "tuples_per_s": n / t}
        out["methods"].append(entry)
        sys.stderr.write(json.dumps(entry) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
