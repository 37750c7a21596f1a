#!/bin/bash
# Session-5 final capture (run under gpurun, 1 GPU), each ncu step only after
# its plain command exited 0:
#  1. smoke() and the full -m gpu suite;
#  2. the default bench line;
#  3. the ncu launch list of the same bench command;
#  4. ncu --set full of one steady Trotter step of the kept schedule, forced by
#     env "$2" (so launch indices are fixed), launches S..S+C-1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2s5z}; F=${2:-"SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=3"}; S=${3:-7}; C=${4:-7}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${T}_gputests.log 2>&1; echo "gpu tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_launch.log 2>&1
echo "bench+launch list rc=$?"
timeout 300 env $F python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1500 env $F ncu --set full --import-source on --clock-control none -k regex:sdb_pass -s $S -c $C -o gpurun_out/${T}_full \
  python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_full.log 2>&1
echo "full rc=$?"
