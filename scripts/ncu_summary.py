#!/usr/bin/env python
"""Summarise one gpu_round.sh capture into profiles/ (tracked).

  python scripts/ncu_summary.py gpurun_out/<tag> <tag>

Writes
  profiles/<tag>_launches.md   per-kernel share of the ncu launch list (and
                               <tag>_fast_launches.md for the FAST-mode list)
                               (gpu__time_duration.sum, cold-cache, serialised)
  profiles/<tag>_ncu_full.md   key `ncu --set full` metrics per captured kernel
  profiles/ncu_summary.json    the same metrics, read by bench.py for
                               roofline.traffic (dram bytes per launch)
  profiles/<tag>_bench.json    the bench line of the same call
"""
from __future__ import annotations

import collections
import csv
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__inst_executed.sum",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def launches(src: str):
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > mv:
            v = float(r[mv].replace(",", "")) * SCALE.get(r[mu], 1.0) * 1e6  # -> us
            t[r[kn].split("(")[0]].append(v)
    return t


def full_metrics(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        m = {}
        for k in METRICS:
            if k in h:
                i = h.index(k)
                try:
                    val = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                m[k] = {"value": val, "unit": units[i]}
        res[name] = m
    return res


def main():
    src, tag = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    for csv_name, out_name, extra in (("launches.csv", "launches", ""),
                                      ("launches_fast.csv", "fast_launches", " --mode fast")):
        lf = os.path.join(src, csv_name)
        if not os.path.exists(lf):
            continue
        t = launches(lf)
        tot = sum(sum(v) for v in t.values())
        lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
                 "Cold-cache, serialised replay of `python bench.py --steps 20 --warmup 3 "
                 f"--no-cpu-baseline --no-extras{extra}`; compare shares, not absolutes.", "",
                 "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | "
                         f"{100 * sum(v) / tot:.1f}% |")
        open(os.path.join(PROF, f"{tag}_{out_name}.md"), "w").write("\n".join(lines) + "\n")
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = {}  # this capture only: no entries from older builds
    md = [f"# {tag}: `ncu --set full` captures", ""]
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        for name, m in full_metrics(rep).items():
            md += [f"## `{name}`", "", "| metric | value | unit |", "|---|---|---|"]
            md += [f"| {k} | {v['value']:g} | {v['unit']} |" for k, v in m.items()]
            md.append("")
            rd = m.get("dram__bytes_read.sum", {})
            wr = m.get("dram__bytes_write.sum", {})
            dram = None
            if rd and wr:
                dram = rd["value"] * SCALE.get(rd["unit"], 1) + wr["value"] * SCALE.get(wr["unit"], 1)
            base = name.split("<")[0].replace("void ", "").strip()
            summ[base] = {"tag": tag, "dram_bytes_per_launch": dram,
                          "metrics": {k: v["value"] for k, v in m.items()}}
    open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w").write("\n".join(md) + "\n")
    json.dump(summ, open(summ_path, "w"), indent=1)
    bj = os.path.join(src, "bench.json")
    if os.path.exists(bj):
        shutil.copy(bj, os.path.join(PROF, f"{tag}_bench.json"))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
