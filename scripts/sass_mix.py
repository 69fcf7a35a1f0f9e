#!/usr/bin/env python
"""Instruction mix + stall samples of one ncu report's SASS page.
usage: python scripts/sass_mix.py <report.ncu-rep> [top]"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
iS, iE = h.index("Source"), h.index("Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
op, st = collections.Counter(), collections.Counter()
hot = []
for x in rows:
    try:
        n = int(x[iE] or 0)
        w = int(x[iW] or 0)
    except (ValueError, IndexError):
        continue
    toks = x[iS].split()
    o = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    o = o.split(".")[0]
    op[o] += n
    st[o] += w
    hot.append((w, x[0], x[iS][:80]))
tot = sum(op.values())
print("total warp-instructions", tot, " stall samples", sum(st.values()))
for k, v in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    print(f"{k:10s} {v:12d} {100 * v / tot:5.1f}%  stall {st[k]}")
print("hottest instructions (stall samples):")
for w, a, s in sorted(hot, reverse=True)[:15]:
    print(w, a, s)
