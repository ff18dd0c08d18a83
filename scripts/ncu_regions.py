#!/usr/bin/env python
"""Aggregate an ncu source page (instructions executed + stall samples) by line ranges.

    python scripts/ncu_regions.py REP.ncu-rep FILE_SUFFIX name:lo-hi [name:lo-hi ...]
"""
import collections
import csv
import subprocess
import sys

rep, suffix, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
regions = [(s.split(":")[0], *map(int, s.split(":")[1].split("-"))) for s in specs]
agg, stl = collections.Counter(), collections.Counter()
hdr, fname, tot, tst = None, None, 0, 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iIE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0] == "":
        continue  # SASS rows: the source row above carries the line's totals
    try:
        ln, ie, ss = int(r[0]), int(r[iIE] or 0), int(r[iS] or 0)
    except ValueError:
        continue
    tot += ie
    tst += ss
    name = "other-file"
    if fname and fname.endswith(suffix):
        name = "other"
        for n, lo, hi in regions:
            if lo <= ln <= hi:
                name = n
                break
    agg[name] += ie
    stl[name] += ss
print(f"{'region':20s} {'instr%':>7s} {'stall%':>7s}")
for n, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{n:20s} {100 * v / max(tot, 1):7.1f} {100 * stl[n] / max(tst, 1):7.1f}")
print(f"total instructions {tot:.4g}, stall samples {tst}")
