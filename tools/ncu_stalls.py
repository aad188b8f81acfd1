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


def reasons(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = {h[i]: 0 for i in cols}
    for r in rows[2:]:
        for i in cols:
            try:
                tot[h[i]] += int(r[i])
            except ValueError:
                pass
    s = sum(tot.values()) or 1
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {k:28s} {v / s:6.3f}")


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "reasons":
    reasons(sys.argv[1])
