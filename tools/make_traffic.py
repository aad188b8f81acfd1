#!/usr/bin/env python
"""Refresh profiles/ncu_traffic.json from the `--set full` summaries under
profiles/r02/ (tools/ncu_summary.py full): traffic = dram__bytes_read.sum +
dram__bytes_write.sum of the captured launch.  The algorithmic bytes and the
kernel descriptions are kept from the existing file."""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(path):
    tot, dur = 0.0, None
    for line in open(path):
        m = re.search(r"dram__bytes_(read|write)\.sum = ([0-9.]+) (\w+)", line)
        if m:
            tot += float(m.group(2)) * UNIT[m.group(3)]
        m = re.search(r"gpu__time_duration\.sum = ([0-9.]+) us", line)
        if m:
            dur = float(m.group(1))
    return int(tot), dur


def main():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tr = json.load(open(p))
    for cfg, classes in tr.items():
        if not isinstance(classes, dict):
            continue
        for cls, e in classes.items():
            cap = e.get("capture", "").split(" ")[0]
            f = os.path.join(ROOT, cap)
            if not cap or not os.path.exists(f):
                print(f"{cfg}/{cls}: capture {cap!r} missing, kept", file=sys.stderr)
                continue
            e["traffic"], e["captured_us"] = dram_bytes(f)
    json.dump(tr, open(p, "w"), indent=1)
    print(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main()
