#!/bin/bash
# Session-5 validation + profiles (run under gpurun, 1 GPU), each ncu step only
# after the plain command exited 0:
#  1. smoke() and the full -m gpu suite;
#  2. the default bench line;
#  3. the ncu launch list of the same bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2s5f}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${T}_gputests.log 2>&1; echo "gpu tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_launch.log 2>&1
echo "bench+launch list rc=$?"
