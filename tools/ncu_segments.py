#!/usr/bin/env python
"""Warp-stall samples and executed instructions between barriers / exits, from an
`ncu -i X.ncu-rep --page source --csv` export: which phase of a kernel holds the
warps (used on k_chol: load | panel | barrier wait + trailing update | substitutions)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
num = lambda v: int(v) if v.isdigit() else 0
tot = sum(num(r[si]) for r in data) or 1
print(f"total samples {tot}")
print(f"{'from':>6} {'to':>6}  {'ends at':32} {'samples':>8} {'share':>6} {'warp instr':>11}")
start, cur, curi = data[0][0][-5:], 0, 0
for r in data:
    cur += num(r[si])
    curi += num(r[ie])
    if "BAR.SYNC" in r[1] or "EXIT" in r[1]:
        print(f"{start:>6} {r[0][-5:]:>6}  {r[1].strip()[:32]:32} {cur:8d} {cur / tot:6.3f} {curi:11d}")
        start, cur, curi = r[0][-5:], 0, 0
print(f"{start:>6} {'end':>6}  {'':32} {cur:8d} {cur / tot:6.3f} {curi:11d}")
top = sorted(data, key=lambda r: -num(r[si]))[:8]
print("top stalled lines:")
for r in top:
    print(f"  {num(r[si]) / tot:6.3f}  {r[0][-5:]}  {r[1].strip()[:80]}")
