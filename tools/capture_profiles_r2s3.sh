#!/bin/bash
# Round-2 profile capture (run under gpurun, 1 GPU), each step only after the
# plain command exited 0:
#  1. the default bench line;
#  2. the ncu launch list of the same bench command (plan-time autotune trials
#     first, then the timed steps);
#  3. one `ncu --set full` capture of a steady-state Trotter step of the
#     autotuned schedule (forced by env so launch indices are fixed: per-term
#     diagonal ops, <= 2 Hadamard levels per pass, TMA), launches 10..19.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
F="SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=2"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/r2s3_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 env $F python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/r2s3_plain.log 2>&1 && \
timeout 1500 env $F ncu --set full --import-source on --clock-control none -k regex:sdb_pass -s 11 -c 10 -o gpurun_out/r2s3_full \
  python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/r2s3_ncu_full.log 2>&1
echo "full rc=$?"
