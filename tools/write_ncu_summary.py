"""Write profiles/r02_ncu_summary.md and profiles/r02_traffic.json from the
captures of tools/profile_round.sh (gpurun_out/: the raw-page CSV exports
prof_<name>.raw.csv, the launch list launches.csv, the default bench line
bench_default.log), here, no GPU needed:

    python tools/write_ncu_summary.py [gpurun_out]

`r02_traffic.json` is what bench.py's roofline reads for `traffic` (DRAM read +
write per launch of each kernel) and `smem_roofline.ncu_wavefronts_per_launch`.
"""

from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "": 1}
CAPS = [("vab", "Bit-sliced VA pass, ids mode: filter (mode 3) + scatter, first pass of the C5 bench batch"),
        ("vac", "Bit-sliced VA pass, count mode (mode 0), first pass of the C5 bench batch"),
        ("colb", "Multi-query columnar ids pass (32 C5 queries) + its expansion"),
        ("col", "Single-query columnar scan, ids mode (C5)"),
        ("va", "Single-query VA scan, count mode (C5)"),
        ("row", "Row-wise scan, count mode (C2)")]


def short(name: str) -> str:
    n = name.split("(VaBatchArgs")[0].split("(mdrq::")[0].split("(BatchArgs")[0].split("(const")[0]
    n = n.replace("void ", "").replace("mdrq::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return n.replace("(int)", "").replace("(bool)", "").strip()


def rows_of(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {k: (v, units[i]) for i, (k, v) in enumerate(zip(hdr, r))}
        out.append(d)
    return out


def num(d, key):
    v, u = d[key]
    return float(str(v).replace(",", "")) * SCALE.get(u, 1)


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    traffic = {"_source": "ncu --set full (tools/profile_round.sh), DRAM read + write per launch; "
                          "profiles/r02_ncu_summary.md", "smem_wavefronts": {}}
    sections = []
    for name, title in CAPS:
        path = os.path.join(src, f"prof_{name}.raw.csv")
        if not os.path.exists(path):
            continue
        sections.append(f"### {title}\n")
        sections.append(ncu_summary.full(path))
        for d in rows_of(path):
            k = short(d["Kernel Name"][0])
            traffic[k] = int(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"))
            if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in d:
                traffic["smem_wavefronts"][k] = int(num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"))
    with open(os.path.join(ROOT, "profiles", "r02_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
        fh.write("\n")
    bench = None
    bl = os.path.join(src, "bench_default.log")
    if os.path.exists(bl):
        bench = json.loads(open(bl).read().strip().splitlines()[-1])
        with open(os.path.join(ROOT, "profiles", "r02_bench_line.json"), "w") as fh:
            json.dump(bench, fh)
            fh.write("\n")
    lines = ["# Round 2 — ncu evidence (C5 workload)", "",
             "Captured with `tools/profile_round.sh` on one B200 (sm_100a), `--clock-control none`, each ncu",
             "command after the same command exited 0 without ncu; launches selected by NVTX range",
             "(`tools/prof_c5.py`: the timed count / ids pass of a prepared batch, after its sizing run).",
             "ncu numbers are cold-cache and serialised: compare shares, not absolutes (bench.py times",
             "with CUDA events on the launching stream).", ""]
    if bench:
        pp = bench["pass_profile"]
        lines += [f"Bench line of the same round (`profiles/r02_bench_line.json`): **{bench['ms_per_step']:.1f} ms per "
                  f"10 000-query C5 step in ids mode = {bench['value']:.3g} tuple-queries/s**, count mode "
                  f"{bench['modes']['count']['ms_per_step']:.1f} ms; pass profile (ids): filter "
                  f"{pp['scan']['ms']:.1f} ms, scatter + block lists + unpermute {pp['id_write']['ms']:.1f} ms, "
                  f"scans {pp['compaction']['ms']:.2f} ms; e2e (`VaFile.search_stream`, 20 GB of ids per step "
                  f"to pinned host memory) {bench['e2e']['ms_per_step']:.0f} ms per step.", ""]
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        lines += ["## Launch list — `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-paths --no-e2e`",
                  "", ncu_summary.launches(lp), ""]
    lines += ["## Full-set captures", ""] + sections
    with open(os.path.join(ROOT, "profiles", "r02_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("wrote profiles/r02_ncu_summary.md, r02_traffic.json" + (", r02_bench_line.json" if bench else ""))


if __name__ == "__main__":
    main()
