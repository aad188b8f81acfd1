#!/usr/bin/env python
"""Top stalled SASS lines (warp stall sampling) from an `ncu --page source --csv` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si]) for r in data if r[si].isdigit()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total samples {tot}")
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]:
    print(f"{int(r[si]) / tot:6.3f}  {r[0][-5:]}  {r[1].strip()[:100]}")
