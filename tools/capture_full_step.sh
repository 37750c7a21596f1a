#!/bin/bash
# ncu --set full of launches S..S+C-1 of the config-4 bench with the per-term
# schedule forced (fixed launch indices), after the plain command exits 0.
#   tools/capture_full_step.sh TAG [S] [C] [extra env...]
cd "$(dirname "$0")/.."
tag=$1; s=${2:-11}; c=${3:-3}; shift 3
F="SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=2 $*"
timeout 300 env $F python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1500 env $F ncu --set full --import-source on --clock-control none -k regex:sdb_pass -s $s -c $c -o gpurun_out/${tag}_full \
  python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${tag}_ncu.log 2>&1
echo "full rc=$?" >> gpurun_out/${tag}_ncu.log
