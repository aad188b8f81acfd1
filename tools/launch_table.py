"""Print the per-launch table (duration, grid, kernel) of an ncu
--metrics gpu__time_duration.sum[,launch__grid_size] CSV; `--tail N` keeps
the last N launches (one timed sweep), `--sum` groups them by kernel."""
import collections
import csv
import sys


def load(path):
    hdr, by = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = by.setdefault(d["ID"], {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = d["Metric Value"]
    return list(by.values())


def main():
    path = sys.argv[1]
    tail = int(sys.argv[sys.argv.index("--tail") + 1]) if "--tail" in sys.argv else 0
    L = load(path)[-tail:] if tail else load(path)
    if "--sum" in sys.argv:
        agg = collections.OrderedDict()
        for d in L:
            k = d["name"].split("(")[0][:90]
            a = agg.setdefault(k, [0.0, 0])
            a[0] += float(d["gpu__time_duration.sum"]) / 1e3
            a[1] += 1
        tot = sum(a[0] for a in agg.values())
        for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
            print(f"{us:10.1f} us {100 * us / tot:5.1f}% x{n:3d}  {k}")
        print(f"{tot:10.1f} us total, {len(L)} launches")
        return
    for d in L:
        print(f"{float(d['gpu__time_duration.sum']) / 1e3:9.1f} us grid {d.get('launch__grid_size', ''):>8} "
              f"{d['name'][:100]}")


if __name__ == "__main__":
    main()
