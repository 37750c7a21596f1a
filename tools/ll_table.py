"""Per-launch table of an ncu --csv launch list: python tools/ll_table.py CSV [CSV...]"""
import csv
import sys

for f in sys.argv[1:]:
    lines = [l for l in open(f) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    d = {}
    for r in rows[1:]:
        d.setdefault(int(r[h.index("ID")]), {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    ms = [d[k]["gpu__time_duration.sum"] / 1e6 for k in sorted(d)]
    print(f, "launches", len(ms))
    print("  ms:", " ".join(f"{x:.2f}" for x in ms))
    if "dram__bytes_read.sum" in d[0]:
        print("  DRAM GB:", " ".join(f"{(d[k]['dram__bytes_read.sum'] + d[k]['dram__bytes_write.sum']) / 1e9:.1f}" for k in sorted(d)))
