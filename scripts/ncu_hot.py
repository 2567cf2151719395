#!/usr/bin/env python
"""Hot SASS lines of one kernel in an ncu report (executed count, stall samples):
    python scripts/ncu_hot.py report.ncu-rep [frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, d = rows[1], rows[2:]
ia, isrc, ist = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia] or 0) for r in d)
sm = sum(int(r[ist] or 0) for r in d)
print("total warp instructions", tot, "stall samples", sm)
mx = max(int(r[ia] or 0) for r in d)
for i, r in enumerate(d):
    c, s = int(r[ia] or 0), int(r[ist] or 0)
    if c > mx * 0.3 or s > sm * frac:
        print(f"{i:5d} {c:11d} {100.0 * s / sm:5.1f}% {r[isrc][:90]}")
