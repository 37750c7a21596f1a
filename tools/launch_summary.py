"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launch count, total / mean device time and share."""
import collections
import csv
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"].split("(")[0], r["Grid Size"], r["Block Size"], float(r["Metric Value"])))
    tot = sum(r[3] for r in rows)
    agg = collections.OrderedDict()
    for name, g, b, ns in rows:
        k = (name, g, b)
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + ns)
    print(f"{'kernel':50s} {'grid':>12s} {'block':>12s} {'n':>5s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for (name, g, b), (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:50]:50s} {g:>12s} {b:>12s} {c:5d} {s / 1e6:10.3f} {s / c / 1e6:9.3f} {100 * s / tot:5.1f}%")
    print(f"total {len(rows)} launches, {tot / 1e6:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
