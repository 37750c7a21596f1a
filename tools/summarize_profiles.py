"""Turns a capture_profiles.sh run into committed summaries under profiles/:
launch table, ncu full metrics per launch, and the traffic JSON bench.py reads."""
import csv
import io
import json
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
rep = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/{tag}_full.ncu-rep"
source = sys.argv[3] if len(sys.argv) > 3 else "ncu --set full, tools/profile_pass.py 4 30 1 (config 4, n=30)"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
col = lambda name: h.index(name)
launches = []
for r in rows[2:]:
    d = {k: r[col(k)] for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                                "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread")
         if k in h}
    launches.append(d)
units = {k: rows[1][col(k)] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum") if k in h}
def to_bytes(v, u):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
per = [to_bytes(l["dram__bytes_read.sum"], units["dram__bytes_read.sum"]) +
       to_bytes(l["dram__bytes_write.sum"], units["dram__bytes_write.sum"]) for l in launches]
alg = 32.0 * 2 ** 30
summary = {"source": f"{source}, launches 0-{len(launches) - 1} of the capture",
           "algorithmic_bytes_per_launch": alg, "dram_bytes_per_launch": sum(per) / len(per),
           "dram_over_algorithmic": sum(per) / len(per) / alg,
           "launches": [dict(l, dram_bytes=b) for l, b in zip(launches, per)], "units": units}
json.dump(summary, open("profiles/ncu_tile_pass_summary.json", "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "launches"}, indent=1))
