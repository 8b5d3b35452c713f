#!/usr/bin/env python
"""Benchmark of the MDRQ scan hot path (BASELINE.json metric: tuples
scanned/s and achieved HBM GB/s per GPU at 1/2/4/8 B200).

Workload: BASELINE.json configs[4] (C5), the configuration the metric is
quoted on -- n = 5e8 tuples, m = 10, float32 uniform [0, 1) from
default_rng(0) (the reference's gen_uniform, generated chunk-parallel,
bit-identical), one batch of 10 000 full-match queries at selectivity 1e-3
(width 0.001**(1/10), lower bounds U[0, 1-w) from default_rng(1);
workload.c5_queries) evaluated in multi-query passes.  One STEP = the whole
10 000-query batch over the device-resident table in ids mode (ascending
uint32 ids per query + offsets, ~5e9 ids = 20 GB); the count-only mode of the
same batch is measured beside it (``modes.count``).

``value`` = tuple-query evaluations per second = n x queries / step time
(every query is decided for every tuple; the unit the reference's CPU scan is
measured in by ``--impl reference``).  ``tuples_per_s`` (= n x HBM passes /
t) and ``queries_per_s`` are reported beside it.

With N > 1 (torchrun, one rank per GPU) the SAME 5e8-row table is split into
N contiguous row shards (strong scaling): rank r generates and
holds rows shard_range(n, N, r) with global ids, scans them, and the step
ends with the NCCL all_gather of the per-query counts (every rank learns the
global result offsets); the full id exchange and the per-rank direct copy
of each rank's ids into one host buffer are timed separately.

``--impl reference`` times the reference's own CPU scan (the reference's
compiled ``scan_rows`` from oracle/_ref driven like HorizontalScan, all host
threads) on a bounded sample of the same queries over the same table.
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import shutil
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N_TOTAL = 500_000_000
M = 10
SELECTIVITY = 1e-3
NQ = 10_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto")
    ap.add_argument("--no-paths", action="store_true",
                    help="skip the per-path cost table, the columnar roofline probe and the C2 line")
    ap.add_argument("--force-merge", action="store_true",
                    help="run the NCCL combine even with one rank (torchrun --nproc-per-node 1)")
    ap.add_argument("--merge-in-step", action="store_true",
                    help="include the full id exchange (all ids on every rank) in the timed step")
    ap.add_argument("--n", type=int, default=N_TOTAL, help="tuples in the whole table (split over ranks)")
    ap.add_argument("--queries", type=int, default=NQ)
    ap.add_argument("--count-steps", type=int, default=None, help="timed steps of the count-mode batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-host-gather", action="store_true",
                    help="skip the per-rank direct copy of the merged ids into one shared host buffer")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.exe = shutil.which("nvidia-smi")

    def _run_nvml(self) -> bool:
        """NVML directly (sub-millisecond queries): a sample every ~2 ms, so a
        timed region of a few tens of ms still gets a median; False when NVML
        is unavailable (then nvidia-smi, ~10 samples/s)."""
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            return False
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        try:
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.002)
        finally:
            try:
                nv.nvmlShutdown()
            except Exception:
                pass
        return True

    def _run(self):
        if self._run_nvml() or not self.exe:
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run([self.exe, "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU legs --

def cpu_reference_rate(values, lo, hi, budget_s: float, threads: int, max_queries: int | None = None):
    """The reference's HorizontalScan on the host (oracle/_ref kernels, or the
    C restatement when that build is absent).  Returns (tuples/s, kind,
    queries timed, threads, seconds)."""
    import oracle
    scan = oracle.ReferenceHorizontalScan(values, threads=threads, seed=0)
    try:
        n = values.shape[0]
        t0 = time.perf_counter()
        scan.search(lo[0], hi[0])   # warm
        first = time.perf_counter() - t0
        nq = max(1, min(int(budget_s / max(first, 1e-6)), lo.shape[0]))
        if max_queries:
            nq = min(nq, max_queries)
        t0 = time.perf_counter()
        acc = 0
        for i in range(nq):
            acc += scan.search(lo[i], hi[i]).size
        dt = time.perf_counter() - t0
        return n * nq / dt, scan.kind, nq, scan.threads, dt
    finally:
        scan.close()


def load_workload(n: int, nq: int, world: int, rank: int):
    """This rank's contiguous shard of the C5 table (global row ids
    [start, stop)) and the query batch."""
    from paper_1801_03644_b200 import workload
    from paper_1801_03644_b200.parallel import shard_range
    start, stop = shard_range(n, world, rank)
    workers = max(1, (os.cpu_count() or 1) // world)
    t = time.perf_counter()
    values = workload.c5_data(start, stop, n=n, workers=workers)
    gen_s = time.perf_counter() - t
    lo, hi = workload.c5_queries(count=nq)
    return values, start, stop, lo, hi, gen_s


def workload_name(n, nq, world):
    return (f"C5 (BASELINE.json configs[4]): n={n} m={M} float32 uniform seed 0, one batch of {nq} full-match "
            f"queries at selectivity {SELECTIVITY:g} per step, ids mode (ascending uint32 ids per query)"
            + (f", rows sharded over {world} GPUs" if world > 1 else ""))


def run_reference(args):
    """The reference's own CPU scan (oracle/_ref: its compiled scan_rows,
    driven like HorizontalScan over all host threads) on the same C5 table
    and queries; each step a bounded sample of the batch."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    values, _, _, lo, hi, gen_s = load_workload(args.n, args.queries, 1, 0)
    n = values.shape[0]
    threads = os.cpu_count() or 1
    import oracle
    scan = oracle.ReferenceHorizontalScan(values, threads=threads, seed=0)
    try:
        t0 = time.perf_counter()
        scan.search(lo[0], hi[0])
        per_q = time.perf_counter() - t0
        # each step a bounded sample: <= 6 s, and the whole run <= ~2.5 minutes
        step_budget = min(6.0, 150.0 / max(1, args.steps + args.warmup))
        q_per_step = max(1, min(args.queries, int(step_budget / max(per_q, 1e-6))))
        qi = 1
        for _ in range(args.warmup):
            for _ in range(q_per_step):
                scan.search(lo[qi % args.queries], hi[qi % args.queries])
                qi += 1
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for _ in range(q_per_step):
                scan.search(lo[qi % args.queries], hi[qi % args.queries])
                qi += 1
            times.append(time.perf_counter() - t0)
        kind = scan.kind
    finally:
        scan.close()
    step = float(np.mean(times))
    value = n * q_per_step / step
    line = {
        "impl": "reference", "metric": "tuple_queries_per_s", "value": value, "unit": "tuple-queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(n, args.queries, 1), "queries_per_step": q_per_step,
                   "same_config": "same table and query batch; each step a bounded sample of its queries",
                   "parallelism": f"host threads={threads}"},
        "queries_per_s": q_per_step / step,
        "cpu_baseline": {"value": value, "unit": "tuple-queries/s", "cores": threads, "kind": kind,
                         "sample": f"{q_per_step} of the {args.queries} queries per step over all {n} tuples"},
        "e2e": {"value": value, "unit": "tuple-queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": {"generate": round(gen_s, 2)},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg --

def timed(fn, steps, stream, world):
    """Device time per call of fn over `steps` calls (CUDA events on the
    launching stream, barrier + synchronize on both sides, max over ranks)."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1801_03644_b200 as eng
    from paper_1801_03644_b200 import _lib

    world, rank, local = dist_env()
    # the NCCL merge runs whenever there is more than one rank; --force-merge
    # exercises it with a single torchrun rank
    merge = world > 1 or args.force_merge
    if merge:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    n_total = args.n
    values, start, stop, lo, hi, t_gen = load_workload(n_total, args.queries, world, rank)
    n = stop - start
    nq = lo.shape[0]
    layouts = _lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE
    t_build = time.perf_counter()
    store = eng.DeviceStore(values, layouts=layouts, va_bits=8, device=dev, id_base=start)
    t_build = time.perf_counter() - t_build
    # a dedicated stream: the library launches on it and the CUDA events are
    # recorded on it
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0

    t_prep = time.perf_counter()
    batch = store.prepare(lo, hi, args.path)
    t_prep = time.perf_counter() - t_prep
    binfo = batch.info()
    total_local = batch.reserve()
    launches_ids = batch.launches(ids=True)
    launches_count = batch.launches(ids=False)
    d_counts = torch.empty(nq, dtype=torch.int64, device=dev)

    def exchange():
        # every rank's ids of every query, rank-ordered (NCCL all_gather of
        # the padded id slices + one segmented-copy kernel)
        d_ids, d_offs, tot = batch.result_device()
        ids_t = _wrap(d_ids, tot, torch.int32, dev)
        offs_t = _wrap(d_offs, nq + 1, torch.int64, dev)
        return eng.combine_ids(offs_t, ids_t)

    def step_ids():
        batch.ids_async(sptr)
        if merge:
            if args.merge_in_step:
                exchange()
            else:
                # the counts combine: every rank learns the global offsets
                # (where its rank-ordered slices go); the id exchange itself
                # is timed separately below
                _, d_offs, _ = batch.result_device()
                offs_t = _wrap(d_offs, nq + 1, torch.int64, dev)
                eng.combine_counts(offs_t[1:] - offs_t[:-1])

    def step_count():
        batch.count_async(d_counts.data_ptr(), sptr)
        if merge:
            eng.combine_counts(d_counts)

    for _ in range(args.warmup):
        step_ids()
    with ClockSampler(dev) as clocks:
        ms = timed(step_ids, args.steps, stream, world)
    for _ in range(2):
        step_count()
    count_steps = args.count_steps or max(3, min(args.steps, 10))
    with ClockSampler(dev) as clocks_count:
        ms_count = timed(step_count, count_steps, stream, world)
    passes = binfo["passes"]
    value = n_total * nq / (ms / 1e3)
    total_ids = total_local
    if merge:
        tt = torch.tensor([total_local], device="cuda", dtype=torch.int64)
        dist.all_reduce(tt)
        total_ids = int(tt.item())

    # ---- the id exchange on its own (all ids of every query on every rank)
    xchg = None
    if merge and not args.merge_in_step:
        exchange()
        xms = timed(exchange, 3, stream, world)
        torch.cuda.empty_cache()   # the exchange's buffers (every rank's ids) before the e2e pools
        xchg = {"ms_per_step": xms, "ids_total": total_ids, "bytes_in_per_rank": 4 * (total_ids - total_local),
                "included_in_value": False,
                "how": "NCCL all_gather of every rank's padded id slices + mdrq_copy_segments placement; "
                       "the step itself ends with the counts combine (global offsets on every rank)"}

    # ---- the ids to the host without an NCCL exchange: every rank writes its
    # own slices into ONE node-shared pinned host buffer at the rank-ordered
    # offsets (its own PCIe link; parallel.gather_ids_to_host)
    host_gather = None
    if merge and not args.no_host_gather:
        host_gather = measure_host_gather(batch, nq, total_ids, total_local, dev, world)

    # ---- dominant kernel of the step: one ids pass with events between
    # launch groups (mdrq_batch_profile), bytes from the kernels' counters
    peak, peak_kind = measured_peaks()
    prof = batch.profile(ids=True, stream=sptr)
    stats = store.stats(nq)
    roofline = roofline_of(binfo["path"], prof, stats, n, nq, total_local, peak, peak_kind)
    if binfo["path"] == "vafile_batch":
        lw = vb_lw(min(nq, 1024), binfo["max_union_dims"])
        key = (f"va_batch_kernel<3, {binfo['max_union_dims']}, {lw}>" if roofline["class"] == "scan"
               else "vb_scatter_kernel")
        roofline.update(ncu_traffic(key))
    rpeak = read_peak(dev)
    add_peaks(roofline, rpeak)
    prof_count = batch.profile(ids=False, stream=sptr)
    stats_count = store.stats(nq)
    roof_count = roofline_of(binfo["path"], prof_count, stats_count, n, nq, 0, peak, peak_kind)
    if binfo["path"] == "vafile_batch" and roof_count["class"] == "scan":
        roof_count.update(ncu_traffic(f"va_batch_kernel<0, {binfo['max_union_dims']}, "
                                      f"{vb_lw(min(nq, 1024), binfo['max_union_dims'])}>"))
    add_peaks(roof_count, rpeak)

    # ---- the single-query columnar scan kernel (HBM-bound by design), same
    # data, and the per-path cost table; skipped with --no-paths
    col_roof = None
    paths = {}
    c2 = None
    if not args.no_paths:
        col_q = min(nq, 20)
        cb = store.prepare(lo[:col_q], hi[:col_q], "columnar")
        cb.reserve()
        cprof = cb.profile(ids=True, stream=sptr)
        cstats = store.stats(col_q)
        col_roof = roofline_of("columnar", cprof, cstats, n, col_q, None, peak, peak_kind)
        col_roof.update(ncu_traffic("col_scan_kernel<1>"))
        add_peaks(col_roof, rpeak)
        cb.close()
        for p, q in (("vafile_batch", nq), ("columnar_batch", min(nq, 1024)), ("vafile", min(nq, 16)),
                     ("columnar", min(nq, 16))):
            pb = store.prepare(lo[:q], hi[:q], p)
            entry = {"queries": q}
            for mode in ("count", "ids"):
                if mode == "ids":
                    pb.reserve()
                pr = pb.profile(ids=(mode == "ids"), stream=sptr)
                entry[f"{mode}_us_per_query"] = round(sum(v[0] for v in pr.values()) * 1e3 / q, 2)
            paths[p] = entry
            pb.close()
        # wall time of one reference-API call per query (search() / count():
        # host bounds in, int64 ResultSet / count out, one synchronous C call)
        from paper_1801_03644_b200.core import ResultSet
        for p in ("vafile", "columnar"):
            q = min(nq, 8)
            ResultSet(store.ids64(lo[:1], hi[:1], p)[1])
            t0 = time.perf_counter()
            for i in range(q):
                ResultSet(store.ids64(lo[i:i + 1], hi[i:i + 1], p)[1])
            paths[p]["search_wall_us"] = round((time.perf_counter() - t0) * 1e6 / q, 1)
            t0 = time.perf_counter()
            for i in range(q):
                int(store.count(lo[i:i + 1], hi[i:i + 1], p)[0])
            paths[p]["count_wall_us"] = round((time.perf_counter() - t0) * 1e6 / q, 1)

    # ---- e2e through the public API: host queries in, host ids out (pinned).
    # DeviceStore.ids_stream over K steps (the same batch each step): every
    # step builds + uploads its descriptors and copies its ids and offsets to
    # pinned host memory; step k's copy overlaps step k+1's scan.
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(store, lo, hi, args, total_local, nq, n_total, world, stream)

    # ---- C2 beside it (BASELINE.json configs[1], 1000 queries at 1e-3)
    if not args.no_paths and world == 1:
        batch.close()
        c2 = measure_c2(eng, _lib, dev, stream, args.steps, args.warmup)

    cpu = None
    ref_methods = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, kind, qn, thr, dt = cpu_reference_rate(values, lo, hi, budget_s=15.0,
                                                     threads=os.cpu_count() or 1)
        ref_methods = reference_methods()
        cpu = {"value": rate, "unit": "tuple-queries/s", "cores": thr, "kind": kind,
               "sample": f"{qn} of the {nq} queries over all {n} tuples ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": "tuple_queries_per_s", "value": value, "unit": "tuple-queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(n_total, nq, world),
                       "path": binfo["path"], "requested_path": args.path, "passes_per_step": passes,
                       "queries_per_step": nq, "ids_per_step": total_ids,
                       "l2": "inputs (20 GB columns + 5 GB code planes in total) larger than L2 (126 MB); "
                             "no flush",
                       "parallelism": f"contiguous row shards x{world}",
                       "combine": ("none (one rank)" if not merge else
                                   "ids exchanged in the step" if args.merge_in_step else
                                   "counts all_gather in the step; id exchange timed separately (id_exchange)")},
            "tuples_per_s": n_total * passes / (ms / 1e3),
            "queries_per_s": nq / (ms / 1e3),
            "hbm_gbs_per_gpu": roofline["achieved"],
            "roofline": roofline,
            "smem_roofline": smem_roofline(binfo, prof, n, nq, clocks.summary()),
            "modes": {
                "ids": {"value": value, "ms_per_step": ms, "queries_per_s": nq / (ms / 1e3),
                        "gpu_launches_per_step": launches_ids},
                "count": {"value": n_total * nq / (ms_count / 1e3), "ms_per_step": ms_count,
                          "steps": count_steps, "queries_per_s": nq / (ms_count / 1e3),
                          "gpu_launches_per_step": launches_count, "roofline": roof_count,
                          "smem_roofline": smem_roofline(binfo, prof_count, n, nq, clocks_count.summary()),
                          "clocks": clocks_count.summary()},
            },
            "columnar_scan_roofline": col_roof,
            "pass_profile": {k: {"ms": round(v[0], 4), "launches": v[1]} for k, v in prof.items()},
            "pass_profile_count": {k: {"ms": round(v[0], 4), "launches": v[1]} for k, v in prof_count.items()},
            "paths_us_per_query": paths,
            "e2e": e2e,
            "id_exchange": xchg,
            "host_gather": host_gather,
            "c2": c2,
            "gpu_launches": launches_ids * args.steps,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "reference_methods": ref_methods,
            "setup_s": {"generate": round(t_gen, 2), "store_build": round(t_build, 2),
                        "prepare_batch": round(t_prep, 3)},
        }
        print(json.dumps(line), flush=True)
    if not (not args.no_paths and world == 1):
        batch.close()
    store.close()
    if merge:
        dist.destroy_process_group()
    return 0


def measure_host_gather(batch, nq, total_ids, total_local, dev, world):
    """Wall time of parallel.gather_ids_to_host (counts all_gather + every
    rank's placement kernel into the shared pinned buffer + barrier), max over
    ranks; skipped when /dev/shm cannot hold the merged result."""
    import torch
    from paper_1801_03644_b200.parallel import SharedHostBuffer, gather_ids_to_host
    need = 4 * total_ids
    try:
        st = os.statvfs("/dev/shm")
        free = st.f_bavail * st.f_frsize
    except OSError:
        free = 0
    ok = torch.tensor([1 if free > need * 1.05 + (1 << 30) else 0], device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if not int(ok.item()):
        return {"skipped": f"/dev/shm holds {free / 1e9:.1f} GB, the merged ids need {need / 1e9:.1f} GB"}
    d_ids, d_offs, tot = batch.result_device()
    ids_t = _wrap(d_ids, tot, torch.int32, dev)
    offs_t = _wrap(d_offs, nq + 1, torch.int64, dev)
    buf = SharedHostBuffer(need, None, device=dev)
    try:
        o, i, _ = gather_ids_to_host(offs_t, ids_t, None, out=buf)   # warm (also touches the pages)
        assert int(o[-1]) == total_ids
        del o, i
        res = {}
        for method in ("dma", "kernel"):
            t0 = time.perf_counter()
            reps = 2
            for _ in range(reps):
                o, i, _ = gather_ids_to_host(offs_t, ids_t, None, out=buf, method=method)
                del o, i
            res[method] = max_over_ranks((time.perf_counter() - t0) / reps, world)
    finally:
        buf.close()
    dt = res["dma"]
    return {"ms_per_step": dt * 1e3, "bytes_per_rank": 4 * total_local, "ids_total": total_ids,
            "gbs_per_rank": 4 * total_local / dt / 1e9, "kernel_ms_per_step": res["kernel"] * 1e3,
            "how": "counts all_gather, then every rank copies its slices into one POSIX-shared host buffer "
                   "registered with CUDA at the rank-ordered offsets (one DMA copy per query segment; "
                   "kernel_ms_per_step: the placement kernel writing through the mapping instead), barrier; "
                   "wall clock"}


def measure_e2e(store, lo, hi, args, total_local, nq, n_total, world, stream):
    """e2e through the reference-facing API: the VA-file access method over
    this store (what build_method("vafile") returns) answers K repetitions of
    the batch with ``search_stream`` -- per step the RangeQuery batch is
    stacked and its bounds go host->device, the planner runs the sorted
    multi-query passes, and the step's ids + offsets come back into pinned
    host memory; step k's copy overlaps step k+1's device pass."""
    import torch
    import torch.distributed as dist
    from paper_1801_03644_b200 import workload
    from paper_1801_03644_b200.vafile import VaFile
    method = VaFile(store, None)
    queries = workload.queries_from_arrays(lo, hi)
    ids_bytes = int(total_local * 4 + (nq + 1) * 8)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    nbuf = 2 if avail > 3 * (total_local * 4 + (1 << 30)) * world else 1
    t0 = time.perf_counter()
    pinned = [torch.empty(max(1, total_local + 1024), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
              for _ in range(nbuf)]
    pin_s = time.perf_counter() - t0
    e2e_steps = max(3, min(args.steps, 20))   # the first step's device pass is the only unhidden part
    # warm: every slot of the stream (3) sizes its buffers once (the first two
    # batches of a store's first stream leave raw -- no result size is known
    # yet --, the next three allocate every slot's packed-copy staging)
    method.search_stream([queries] * 5, outs=[pinned[k % nbuf] for k in range(5)])
    if world > 1:
        dist.barrier()
    info = {}
    t0 = time.perf_counter()
    res = method.search_stream([queries] * e2e_steps, outs=[pinned[k % nbuf] for k in range(e2e_steps)], info=info)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    assert all(int(r.offsets[-1]) == total_local for r in res), "stream result differs from the timed batch"
    # the last step's ids, rebuilt on the host from the packed copy, against
    # the device result of the timed batch (count + set hash per query is
    # the tests' job; here: the copy that was timed is the right one)
    last = res[-1]
    head = min(nq, 64)
    dev_offs, dev_ids = store.ids(lo[:head], hi[:head], "columnar_batch" if head >= 4 else "columnar")
    assert np.array_equal(last.offsets[: head + 1], dev_offs), "stream offsets differ"
    assert np.array_equal(np.asarray(last.ids)[: dev_ids.size], dev_ids), "stream ids differ from the columnar scan's"
    del res, last, dev_ids
    h2d = info.get("h2d_bytes", 0) // e2e_steps   # the batch's descriptors: bounds, query-mask tables, order
    d2h = info.get("d2h_bytes", 0) // e2e_steps or ids_bytes
    packed = info.get("packed_batches", 0)
    # the same stream with the packing off: the raw uint32 ids cross PCIe
    raw_steps = e2e_steps
    os.environ["MDRQ_STREAM_PACK"] = "0"
    try:
        method.search_stream([queries] * 3, outs=[pinned[k % nbuf] for k in range(3)])   # the slots' own pools
        t0 = time.perf_counter()
        method.search_stream([queries] * raw_steps, outs=[pinned[k % nbuf] for k in range(raw_steps)])
        raw_s = (time.perf_counter() - t0) / raw_steps
    finally:
        del os.environ["MDRQ_STREAM_PACK"]
    raw_s = max_over_ranks(raw_s, world)
    store.ids(lo, hi, args.path, out=pinned[0])   # warm
    t0 = time.perf_counter()
    sync_n = 2
    for _ in range(sync_n):
        store.ids(lo, hi, args.path, out=pinned[0])
    sync_s = (time.perf_counter() - t0) / sync_n
    # count-only mode through the same API: one count_batch call per step
    # (bounds host->device, the multi-query count passes, the counts back)
    counts = method.count_batch(queries)   # warm
    assert int(counts.sum()) == total_local, "count_batch differs from the ids total"
    count_n = 5
    t0 = time.perf_counter()
    for _ in range(count_n):
        method.count_batch(queries)
    count_s = max_over_ranks((time.perf_counter() - t0) / count_n, world)
    e2e_s = max_over_ranks(e2e_s, world)
    sync_s = max_over_ranks(sync_s, world)
    # the bound of e2e: this box's pinned device->host bandwidth for one copy
    # of (up to 4 GB of) the step's result
    probe = min(ids_bytes, 4 << 30)
    d_src = torch.empty(probe, dtype=torch.uint8, device="cuda")
    h_dst = torch.from_numpy(pinned[0].view(np.uint8)[:probe])
    d2h_ms = []
    for _ in range(3):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        h_dst.copy_(d_src, non_blocking=True)
        c1.record(stream)
        torch.cuda.synchronize()
        d2h_ms.append(c0.elapsed_time(c1))
    d2h_peak = probe / (min(d2h_ms) / 1e3) / 1e9
    del d_src, h_dst, pinned
    return {"value": n_total * nq / e2e_s, "unit": "tuple-queries/s",
            "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h) * world,
            "result_bytes_per_step": ids_bytes * world,
            "api": f"VaFile.search_stream (the build_method('vafile') object over the bench store): {e2e_steps} "
                   f"repetitions of the RangeQuery batch pipelined (copy of step k under the device pass of step "
                   f"k+1, host unpack of step k-1 beside them), {nbuf} output buffer(s); wall clock, max over ranks",
            "ms_per_step": e2e_s * 1e3,
            "packed_batches": f"{packed} of {e2e_steps}: ids leave the device as 16-bit low halves + per-query "
                              "bucket ends and are rebuilt to uint32 on the host threads (mdrq_unpack_ids16)",
            "packed_share": {"value": info.get("packed_share"),
                             "note": "share of a batch's queries sent packed (the rest raw), steered to the "
                                     "shortest measured step period of the stream"},
            "unpacked": {"ms_per_step": raw_s * 1e3, "value": n_total * nq / raw_s,
                         "note": f"MDRQ_STREAM_PACK=0, {raw_steps} steps: raw uint32 ids over PCIe"},
            "d2h_roofline": {"achieved_gbs": d2h / e2e_s / 1e9, "peak_gbs": d2h_peak,
                             "frac": d2h / e2e_s / 1e9 / d2h_peak,
                             "peak_kind": "measured in this run: one pinned copy of min(result, 4 GB) per GPU"},
            "sync_call": {"value": n_total * nq / sync_s, "ms_per_step": sync_s * 1e3,
                          "api": "DeviceStore.ids into a pinned buffer, one synchronous call per step"},
            "count_call": {"value": n_total * nq / count_s, "ms_per_step": count_s * 1e3,
                           "d2h_bytes_per_step": nq * 8 * world,
                           "api": "VaFile.count_batch (count-only mode), one synchronous call per step"},
            "pin_s": round(pin_s, 2)}


def measure_c2(eng, _lib, dev, stream, steps, warmup):
    """BASELINE.json configs[1] at selectivity 1e-3 (1000 queries, 5e7 x 8),
    the round-1 headline, kept as a secondary number."""
    from paper_1801_03644_b200 import workload
    values = workload.c2_data()
    lo, hi = workload.c2_queries(levels=(1e-3,))[1e-3]
    sptr = stream.cuda_stream
    with eng.DeviceStore(values, layouts=_lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE, va_bits=8, device=dev) as st:
        b = st.prepare(lo, hi, "auto")
        total = b.reserve()
        for _ in range(warmup):
            b.ids_async(sptr)
        ms = timed(lambda: b.ids_async(sptr), steps, stream, 1)
        for _ in range(2):
            b.count_async(0, sptr)
        msc = timed(lambda: b.count_async(0, sptr), steps, stream, 1)
        prof = b.profile(ids=True, stream=sptr)
        b.close()
    n, nq = values.shape[0], lo.shape[0]
    return {"workload": "C2: 5e7 x 8 uniform seed 0, 1000 full-match queries at 1e-3",
            "ids_ms_per_step": ms, "count_ms_per_step": msc, "value": n * nq / (ms / 1e3),
            "unit": "tuple-queries/s", "ids_per_step": total,
            "pass_profile": {k: {"ms": round(v[0], 4), "launches": v[1]} for k, v in prof.items()}}


def vb_lw(nq: int, kb: int) -> int:
    """The LW template argument of the bit-sliced pass's filter kernel
    (vabatch.cu run_kb): 8 / 16 lanes per tuple for passes of <= 256 / 512
    queries, else the four-word layout (128) for unions of <= 10 dims and 32
    for wider ones (MDRQ_VB_WORDS overrides)."""
    if kb > 16:
        return 32
    if nq <= 256:
        return 8
    if nq <= 512:
        return 16
    words = os.environ.get("MDRQ_VB_WORDS") or ("4" if kb <= 10 else "1")
    return {"1": 32, "2": 64}.get(words, 128)


def reference_methods():
    """The reference's own access methods (scan, VA-file, kd-tree, R*-tree)
    through its public API on this host, bounded (tools/reference_methods.py
    bench_leg; the package pip-installed into baseline/_ref by build()), or
    None when it is not installed."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("reference_methods",
                                                  os.path.join(ROOT, "tools", "reference_methods.py"))
    mod = importlib.util.module_from_spec(spec)
    try:
        spec.loader.exec_module(mod)
        return mod.bench_leg()
    except Exception as e:   # the baseline table is informative; never fail the bench on it
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


def smem_roofline(binfo, prof, n, nq, clocks):
    """The resource that bounds the bit-sliced filter pass: shared-memory
    wavefronts.  Algorithmic count per pass: the table row of every tuple
    and union dimension -- 32 lanes x 4 bytes of overlap words (1 wavefront)
    for unions of <= 10 dims, whose candidates are all refined from staged
    values, else 32 x 8 bytes of (overlap, containment) words (2 wavefronts);
    peak: 1 wavefront per cycle per SM at the SM clock measured during the
    timed region (148 SMs)."""
    if binfo["path"] != "vafile_batch" or not prof["scan"][1]:
        return None
    kb = binfo["max_union_dims"]
    wavefronts = (1.0 if kb <= 10 else 2.0) * n * kb
    launch_s = prof["scan"][0] / prof["scan"][1] / 1e3
    mhz = clocks.get("sm_mhz") or 1965.0
    peak = 148 * mhz * 1e6
    achieved = wavefronts / launch_s
    out = {"resource": "shared-memory wavefronts (table rows)", "achieved": achieved, "peak": peak,
           "unit": "wavefronts/s", "frac": achieved / peak, "algo_wavefronts_per_launch": wavefronts,
           "sm_mhz": mhz}
    # all the kernel's smem wavefronts (tables + shuffles + queue + refinement)
    # from the committed ncu capture, over this run's launch time
    key = f"va_batch_kernel<3, {kb}, {vb_lw(nq, kb)}>"
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        with open(f) as fh:
            w = json.load(fh).get("smem_wavefronts", {}).get(key)
        if w:
            out["ncu_wavefronts_per_launch"] = float(w)
            out["frac_all_wavefronts"] = w / launch_s / peak
            out["ncu_source"] = f"{os.path.relpath(f, ROOT)}: smem_wavefronts {key}"
            break
    return out


SPEC_HBM_GBS = 8000.0   # B200 HBM3e spec, the BASELINE roofline denominator


def read_peak(device: int) -> float | None:
    """Measured read-stream bandwidth (mdrq_measure_read_bw: 4 GB, best of
    5), SURVEY.md 8(d)'s second denominator beside the copy peak."""
    import ctypes
    from paper_1801_03644_b200 import _lib
    g = ctypes.c_double(0)
    rc = _lib.load().mdrq_measure_read_bw(device, 4 << 30, 5, ctypes.byref(g))
    return g.value if rc == 0 else None


def add_peaks(roof: dict | None, rpeak: float | None) -> None:
    if not roof:
        return
    roof["peak_spec"] = SPEC_HBM_GBS
    roof["frac_spec"] = roof["achieved"] / SPEC_HBM_GBS
    roof["peak_read_measured"] = rpeak
    roof["frac_read_measured"] = roof["achieved"] / rpeak if rpeak else None


def ncu_traffic(kernel: str) -> dict:
    """DRAM read + write bytes per launch of `kernel` from the newest committed
    ncu --set full capture (profiles/rNN_traffic.json, written from the
    round's tools/profile_round.sh captures); null when not captured."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for f in reversed(files):
        with open(f) as fh:
            d = json.load(fh)
        if kernel in d:
            return {"traffic": float(d[kernel]), "traffic_source": f"{os.path.relpath(f, ROOT)}: {kernel}"}
    return {"traffic": None}


def roofline_of(path, prof, stats, n, nq, total_ids, peak, peak_kind):
    """Roofline of the dominant kernel class of one profiled pass.

    Algorithmic bytes: the HBM bytes the algorithm
    must move -- the column / code-plane loads the scan kernels issue
    (skipped loads are not counted), plus the kernel's own outputs (the
    verdict bitmask n/8 B per query, or the ids 4 B each)."""
    cls = max(("scan", "compaction", "id_write"), key=lambda c: prof[c][0])
    ms, nl = prof[cls]
    nl = max(nl, 1)
    loaded = float(sum(s.bytes_loaded for s in stats))
    ids_bytes = 4.0 * (total_ids or 0)
    if path.endswith("_batch"):
        passes = max(1, prof["scan"][1])
        if cls == "scan":
            # filter pass: the union's code planes (and, for unions of <= 10
            # dims, their exact columns, refined on chip) + (ids mode) one
            # 4-byte staged (tuple, query) record per match
            algo = (loaded + ids_bytes) / passes
        else:
            algo = (2 * ids_bytes) / max(nl, 1)   # records read + ids written
        kernel = {"vafile_batch": "va_batch_kernel (bit-sliced, <=1024 queries/pass)",
                  "columnar_batch": "col_batch_count_kernel (<=32 queries/pass)"}[path]
        kernel += " filter pass" if cls == "scan" else " scatter"
    else:
        algo = (loaded + nq * n / 8.0) / nl
        kernel = {"columnar": "col_scan_kernel", "vafile": "va_scan_kernel", "rowwise": "row_scan_kernel"}[path]
    launch_ms = ms / nl
    achieved = algo / (launch_ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "peak_kind": peak_kind, "kernel": kernel, "class": cls,
            "algo_bytes_per_launch": algo, "launch_ms": launch_ms, "launches": nl,
            "class_share_of_pass": ms / max(1e-9, sum(v[0] for v in prof.values()))}


def _wrap(ptr: int, count: int, dtype, dev):
    """Device pointer -> torch tensor (no copy) via __cuda_array_interface__."""
    import torch
    typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=torch.device("cuda", dev))


if __name__ == "__main__":
    sys.exit(main())
