"""Regenerate profiles/r01_ncu_summary.md and profiles/r01_traffic.json from
the captures of tools/profile_round.sh (gpurun_out/), here, no GPU needed:

    python tools/write_ncu_summary.py [gpurun_out]

Kernel tables come from tools/ncu_summary.py; the bench line is the default
`python bench.py` run of the same round (gpurun_out/bench_default.log).
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

EXTRA = ["l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"]


def raw(path):
    text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[0]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("mdrq::<", "")
        out[short] = {k: r[i] for i, k in enumerate(hdr)}
    return out


def num(x):
    return float(str(x).replace(",", ""))


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    bench = json.loads(open(os.path.join(src, "bench_default.log")).read().strip().splitlines()[-1])
    caps = {k: raw(os.path.join(src, f"prof_{k}.ncu-rep")) for k in ("vab", "col", "va", "row")}
    traffic = {"_source": "ncu --set full, profiles/r01_ncu_summary.md (tools/profile_round.sh), "
                          "DRAM read + write per launch", "smem_wavefronts": {}}
    # ncu prints DRAM bytes in Gbyte / Mbyte: convert with the units row
    for k, cap in caps.items():
        text = subprocess.run(["ncu", "-i", os.path.join(src, f"prof_{k}.ncu-rep"), "--page", "raw", "--csv"],
                              capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(text)))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace(
                "unnamed>::", "").replace("mdrq::<", "")
            rd = num(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = num(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            traffic[name] = int(rd + wr)
            if k == "vab":
                traffic["smem_wavefronts"][name] = int(num(r[hdr.index(
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")]))
    with open(os.path.join(ROOT, "profiles", "r01_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
        fh.write("\n")
    with open(os.path.join(ROOT, "profiles", "r01_bench_line.json"), "w") as fh:
        json.dump(bench, fh)
        fh.write("\n")
    filt = next(v for k, v in caps["vab"].items() if k.startswith("va_batch_kernel"))
    fname = next(k for k in caps["vab"] if k.startswith("va_batch_kernel"))
    pp = bench["pass_profile"]
    lines = [
        "# Round 1 — ncu evidence",
        "",
        "Captured with `tools/profile_round.sh` on one B200 (sm_100a, driver 580.159), `--clock-control none`,",
        "each ncu command after the same command exited 0 without ncu; summarised by",
        "`tools/write_ncu_summary.py`.  ncu numbers are cold-cache and serialised: compare shares, not",
        "absolutes (bench.py times with CUDA events on the launching stream).",
        "",
        f"Bench line of the same round (`profiles/r01_bench_line.json`, `python bench.py`, {bench['steps']} steps "
        f"after {bench['warmup']} warm-up): **{bench['ms_per_step']:.2f} ms/step = {bench['value']:.3g} tuples/s** "
        f"(C2, 5e7 x 8, 1 000 queries at s = 1e-3, ids mode); pass profile: filter {pp['scan']['ms']:.2f} ms, "
        f"scatter + block list {pp['id_write']['ms']:.2f} ms, scans {pp['compaction']['ms']:.2f} ms; e2e through "
        f"`DeviceStore.ids_stream` (host queries in, pinned host ids out, 200 MB per step over PCIe) "
        f"{bench['e2e']['value']:.3g} tuples/s; reference CPU arm (`oracle/_ref`, the reference's compiled "
        f"`scan_rows`, {bench['cpu_baseline']['cores']} threads) {bench['cpu_baseline']['value']:.3g} tuples/s.",
        "",
        "## Launch list — `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-paths`",
        "",
        "`gpu__time_duration.sum` per kernel over the whole command: store build (transpose / encode /",
        "min-max / sample / CUB sort / pick), the read-stream peak probe (`read_stream_kernel`, 6 x 4 GB),",
        "then the batch passes (sizing, warm-up, timed step, profiled pass, the e2e stream and the",
        f"synchronous e2e calls).  The step's kernels are `{fname}` (filter: ids mode, 8-dim union, the",
        "four-word layout) and `vb_scatter_kernel`; `va_batch_kernel<2, 8, 32>` is the recount fallback",
        "(it reads the overflow flag and exits).  Raw CSV: `profiles/r01_launches_bench.csv`.",
        "",
        ncu_summary.launches(os.path.join(src, "launches.csv")),
        "",
        "## Full-set captures",
        "",
        "### Bit-sliced VA filter + scatter (second ids pass of the bench batch)",
        "",
        ncu_summary.full(os.path.join(src, "prof_vab.ncu-rep")),
        "",
        f"Extra counters of the filter: LSU data pipe {num(filt[EXTRA[0]]):.1f} % of peak; smem wavefronts by op: "
        f"ld {num(filt[EXTRA[1]]) / 1e6:.0f} M, st {num(filt[EXTRA[2]]) / 1e6:.0f} M, "
        f"atom {num(filt[EXTRA[3]]) / 1e6:.0f} M.",
        "",
        "Reading: the filter moves 2.0 GB of DRAM per pass (the union's 8 code planes, 0.4 GB, and its 8",
        "exact columns, 1.6 GB, streamed once; + the staged records) = the **algorithmic bytes** (bench",
        "`roofline.algo_bytes_per_launch` 2.2e9 incl. the record writes; `roofline.traffic` is this",
        "capture's read + write, `profiles/r01_traffic.json`) — no re-reads.  It is not HBM-bound: it is",
        "bound by the LSU data pipe (shared-memory wavefronts; 1 per clk per SM) — the table rows alone",
        "are 400 M wavefronts (8 per tuple: 1 024 query bits x 8 dims), the rest the staged cells / values,",
        "the candidate queue and the lane-parallel refinement; bench `smem_roofline` reports both",
        "fractions.  Occupancy is 25 % by design (one CTA of 16 warps per SM; tables, query bounds, staged",
        "values and cells and the queues fill 224 KB).",
        "",
        "The scatter moves the records in and the ids out (the algorithmic volume): one CTA per group sorts",
        "20-block windows in shared memory while the next window's block list and records are in flight.",
        "It is latency-bound (short-scoreboard and barrier stalls), not DRAM-bound: this round its",
        "placement loop lost the per-iteration `S2R SR_CgaCtaId` (shared addresses formed once) and the",
        "10-ballot duplicate match (one ballot per duplicated query): 215 M -> 169 M warp instructions,",
        "0.38 -> 0.33 ms.",
        "",
        "### Single-query columnar scan (`tools/probe_path.py columnar ids 20`, 11th launch)",
        "",
        ncu_summary.full(os.path.join(src, "prof_col.ncu-rep")),
        "",
        "Reading: ~1.03 GB of DRAM in ~161 us = ~6.4 TB/s = ~98 % of the measured copy peak (6.54 TB/s,",
        "`MEASURED_PEAKS.json`), ~90 % of the measured read-stream peak (~7.05 TB/s, `mdrq_measure_read_bw`);",
        "the algorithmic bytes (64-byte blocks with a surviving tuple) are 0.88 GB per launch (bench",
        "`columnar_scan_roofline`).",
        "",
        "### Single-query VA scan (`tools/probe_path.py vafile count 20`, 26th launch)",
        "",
        ncu_summary.full(os.path.join(src, "prof_va.ncu-rep")),
        "",
        "Reading: 0.40 GB of code planes in ~96 us = ~4.2 TB/s; latency / issue-limited (one 7-op SWAR",
        "range test per 4 codes, a vote per pair of planes, every tuple alive after the last dimension",
        "refined exactly).  Before this round's SWAR rewrite, two planes per step and the 32-register",
        "bound: ~102 us and 70 M warp instructions (now 62 M).",
        "",
        "### Row-wise scan (`tools/probe_path.py rowwise count 3`, 2nd launch)",
        "",
        ncu_summary.full(os.path.join(src, "prof_row.ncu-rep")),
        "",
        "Reading: 1.60 GB (the whole row store) in ~233 us = ~6.9 TB/s of DRAM throughput = ~97 % of the",
        "measured read-stream peak — at the HBM roofline (TMA bulk copies, 3 x 32 KB stages, 2 CTAs / SM).",
        "",
    ]
    with open(os.path.join(ROOT, "profiles", "r01_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines))


if __name__ == "__main__":
    main()
