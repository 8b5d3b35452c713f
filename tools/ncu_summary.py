"""Summarise ncu outputs (run here, no GPU needed) into a markdown table.

    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep   (or prof.raw.csv)
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def _csv_rows(text: str):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.reader(io.StringIO("\n".join(lines[start:]))))


def launches(path: str) -> str:
    rows = _csv_rows(open(path).read())
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("mdrq::<unnamed>::", "").replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = ["| kernel | launches | device time (us, serialised, cold) | share |", "|---|---:|---:|---:|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(out)


def raw_rows(path: str):
    """The raw page of a capture: an .ncu-rep (exported here) or the
    .raw.csv tools/profile_round.sh exports on the GPU box."""
    if path.endswith(".csv"):
        text = open(path).read()
    else:
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(text)))


def full(path: str) -> str:
    rows = raw_rows(path)
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        out.append(f"### `{name}`\n")
        out.append("| metric | value |")
        out.append("|---|---:|")
        for key, label in FULL_METRICS:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
