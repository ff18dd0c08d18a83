#!/usr/bin/env python
"""Per-source-line instruction / stall shares of an ncu report (one file), run here (no GPU).

    python scripts/ncu_lines.py REP.ncu-rep FILE_SUFFIX [lo hi]
"""
import csv
import subprocess
import sys

rep, suffix = sys.argv[1], sys.argv[2]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, fname, tot, tst, agg = None, None, 0, 0, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iIE, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) != len(hdr) or r[0] == "":
        continue
    try:
        ln, ie, ss = int(r[0]), int(r[iIE] or 0), int(r[iS] or 0)
    except ValueError:
        continue
    tot += ie
    tst += ss
    if fname and fname.endswith(suffix) and lo <= ln <= hi:
        a = agg.setdefault(ln, [0, 0, r[1].strip()[:90]])
        a[0] += ie
        a[1] += ss
print(f"total instructions {tot:.4g}, stall samples {tst}")
for ln in sorted(agg):
    ie, ss, txt = agg[ln]
    if ie / max(tot, 1) >= 0.001 or ss / max(tst, 1) >= 0.002:
        print(f"L{ln:5d} {100 * ie / tot:5.1f}% {100 * ss / tst:5.1f}%  {txt}")
