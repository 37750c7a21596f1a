"""Summarise an ncu report: per-launch key metrics + SASS opcode mix."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
idx = [h.index(w) if w in h else None for w in want]
units = rows[1]
for k, row in enumerate(rows[2:]):
    print(f"--- launch {k}")
    for w, i in zip(want, idx):
        if i is not None:
            print(f"  {w:75s} {row[i]} {units[i]}")
if len(sys.argv) > 2:
    n = int(sys.argv[2])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--launch-skip",
                          str(n), "--launch-count", "1"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hdr = r[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    op, opw = collections.Counter(), collections.Counter()
    te = tw = 0
    for row in r[2:]:
        try:
            e, w = int(row[iE] or 0), int(row[iW] or 0)
        except (ValueError, IndexError):
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", row[iS])
        if m:
            op[m.group(2)] += e
            opw[m.group(2)] += w
            te += e
            tw += w
    print(f"launch {n}: opcode mix (instr %, stall-sample %)")
    for o, c in op.most_common(18):
        print(f"  {o:10s} {100 * c / te:6.2f} {100 * opw[o] / max(1, tw):6.2f}")
