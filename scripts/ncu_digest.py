#!/usr/bin/env python
"""Digest of one ncu report: key metrics, stall samples, SASS opcode mix.
usage: scripts/ncu_digest.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(p, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for name, unit, val in zip(h, u, v):
    if name in want:
        print(f"{name:80s} {val:>14s} {unit}")
for name, unit, val in zip(h, u, v):
    if "pcsamp_warps_issue_stalled" in name and "not_issued" not in name and val not in ("0", ""):
        print(f"  stall {name.split('stalled_')[1]:30s} {val}")
src = page("source", "--print-source", "sass")
hdr = src[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
agg, tot = collections.Counter(), 0
for r in src[2:]:
    if len(r) <= iE:
        continue
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    n = int(r[iE] or 0)
    agg[o.split(".")[0]] += n
    tot += n
print("  opcode mix:", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in agg.most_common(12)),
      f"(total {tot})")
