"""Compact per-launch table from tools/ncu_summary.py output: python tools/ncu_table.py REPORT"""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, __file__.replace("ncu_table.py", "ncu_summary.py"), sys.argv[1]],
                     capture_output=True, text=True).stdout
keys = {"gpu__time_duration.sum": "ms", "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%", "smsp__inst_executed.sum": "inst",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
        "dram__bytes_read.sum": "rdGB", "dram__bytes_write.sum": "wrGB",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "long",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "short",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "mio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "wait",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "bar",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "lg",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "math"}
rows, cur = [], None
for line in out.splitlines():
    if line.startswith("--- launch"):
        cur = {}
        rows.append(cur)
        continue
    m = re.match(r"\s+(\S+)\s+([\d.]+)\s*(\S*)", line)
    if m and cur is not None and m.group(1) in keys:
        v = float(m.group(2))
        if m.group(3) == "Gbyte":
            pass
        cur[keys[m.group(1)]] = v
cols = list(keys.values())
print("launch " + " ".join(f"{c:>8}" for c in cols))
for i, r in enumerate(rows):
    vals = []
    for c in cols:
        v = r.get(c)
        vals.append(f"{v:8.3g}" if v is not None else "       -")
    print(f"{i:6d} " + " ".join(vals))
