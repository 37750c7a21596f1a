#!/bin/bash
# LOAD/STORE fold validation + A/B (run under gpurun, 1 GPU):
#  1. parity: JIT tests (folds off / default / always), config 4 at n=30 vs oracle/_ref;
#  2. bench A/B on one box: folds off, default (twice), the no-cap schedule forced;
#  3. launch list + ncu --set full of the default bench's kept schedule.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2fold}
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-other-configs"
timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${T}_tests_jit.log 2>&1; echo "jit tests rc=$?"
timeout 600 python -m pytest tests/test_fullsize_oracle_gpu.py -m gpu -q -x -k "cfg4_n30 or cfg3_n28" > gpurun_out/${T}_tests_full.log 2>&1; echo "fullsize rc=$?"
SDB_LOAD_FOLD=0 SDB_STORE_FOLD=0 timeout 600 $B > gpurun_out/${T}_off.json 2> gpurun_out/${T}_off.err; echo "off rc=$?"
timeout 600 $B > gpurun_out/${T}_on.json 2> gpurun_out/${T}_on.err; echo "on rc=$?"
SDB_LOAD_FOLD=0 SDB_STORE_FOLD=0 timeout 600 $B > gpurun_out/${T}_off2.json 2>/dev/null; echo "off2 rc=$?"
timeout 600 $B > gpurun_out/${T}_on2.json 2>/dev/null; echo "on2 rc=$?"
SDB_LOAD_FOLD=2 SDB_STORE_FOLD=2 timeout 600 $B > gpurun_out/${T}_always.json 2>/dev/null; echo "always rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
