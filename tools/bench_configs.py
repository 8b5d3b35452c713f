"""Per-configuration measurements (BASELINE.json configs C1-C5) on one GPU.

    python tools/bench_configs.py [c1 c2 c3 c4 c5] > profiles/r02_configs.json

For every configuration: the table, its queries (the same seeded inputs the
parity tests use), the device time per query of every path in count and ids
mode (mdrq_batch_profile: CUDA events between launch groups), the planner's
choice, and the reference's own compiled scan (oracle/_ref, HorizontalScan
driving, all host threads) on a bounded sample of the queries.  Batch paths
run the full query set; single-query paths a prefix (stated per entry).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load(cfg):
    from paper_1801_03644_b200 import workload
    if cfg == "c1":
        lo, hi = workload.c1_queries()
        return workload.c1_data(), lo, hi, "1e6 x 3 uniform, 1000 queries at 1%"
    if cfg == "c2":
        levels = workload.c2_queries()
        lo = np.concatenate([v[0] for v in levels.values()])
        hi = np.concatenate([v[1] for v in levels.values()])
        return workload.c2_data(), lo, hi, "5e7 x 8 uniform, 5 x 1000 queries at 1e-5..1e-1"
    if cfg in ("c3", "c4"):
        G = np.load(os.path.join(ROOT, "tests", "golden", f"{cfg}.npz"))
        data = workload.c3_data() if cfg == "c3" else workload.c4_data()
        desc = ("1e8 x 16 Gaussian mixture, 2000 partial-match queries (2-8 dims, 1e-3..5e-2)" if cfg == "c3"
                else "1e7 x 19 genomics-shaped, 5000 partial-match queries (3-5 dims, equality on categoricals)")
        return data, G["lo"], G["hi"], desc
    if cfg == "c5":
        lo, hi = workload.c5_queries()
        return workload.c5_data(), lo, hi, "5e8 x 10 uniform (20 GB), 10000 queries at 1e-3"
    raise ValueError(cfg)


def measure(cfg):
    import torch
    import oracle
    import paper_1801_03644_b200 as eng
    from paper_1801_03644_b200 import _lib
    values, lo, hi, desc = load(cfg)
    n, m = values.shape
    nq = lo.shape[0]
    layouts = _lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE | (_lib.LAYOUT_ROWWISE if n * m * 4 < 8e9 else 0)
    t0 = time.perf_counter()
    st = eng.DeviceStore(values, layouts=layouts, va_bits=8)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    out = {"config": cfg, "workload": desc, "n": n, "m": m, "queries": nq, "store_build_s": round(build_s, 2),
           "paths": {}}
    planner = st.prepare(lo, hi, "auto")
    out["planner_path"] = planner.info()["path"]
    planner.close()
    paths = ["vafile_batch", "columnar_batch", "vafile", "columnar"] + (["rowwise"] if layouts & 2 else [])
    for p in paths:
        q = nq if p.endswith("_batch") else min(nq, 64 if n >= 1e8 else 200)
        b = st.prepare(lo[:q], hi[:q], p)
        entry = {"queries_timed": q}
        for mode in ("count", "ids"):
            if mode == "ids":
                total = b.reserve()
                entry["ids_per_query"] = total / q
            pr = b.profile(ids=(mode == "ids"), stream=sp)
            ms = sum(v[0] for v in pr.values())
            entry[f"{mode}_us_per_query"] = round(ms * 1e3 / q, 2)
            entry[f"{mode}_tuples_per_s"] = n * q / (ms / 1e3)
        out["paths"][p] = entry
        b.close()
    # the reference's compiled scan on the host, bounded sample
    thr = os.cpu_count() or 1
    scan = oracle.ReferenceHorizontalScan(values, threads=thr, seed=0)
    try:
        t0 = time.perf_counter()
        scan.search(lo[0], hi[0])
        first = time.perf_counter() - t0
        k = max(1, min(nq, int(8.0 / max(first, 1e-6))))
        t0 = time.perf_counter()
        for i in range(k):
            scan.search(lo[i], hi[i])
        dt = time.perf_counter() - t0
        out["cpu_reference"] = {"kind": scan.kind, "threads": thr, "queries": k,
                                "us_per_query": round(dt * 1e6 / k, 1), "tuples_per_s": n * k / dt}
    finally:
        scan.close()
    best = min(v.get("ids_us_per_query", 1e30) for v in out["paths"].values())
    out["best_ids_speedup_vs_cpu"] = out["cpu_reference"]["us_per_query"] / best
    st.close()
    return out


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    res = []
    for c in cfgs:
        r = measure(c)
        res.append(r)
        sys.stderr.write(json.dumps(r) + "\n")
        sys.stderr.flush()
    print(json.dumps(res, indent=1))
