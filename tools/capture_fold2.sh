#!/bin/bash
# Session-6 capture after the LOAD/STORE folds (run under gpurun, 1 GPU), each
# ncu step only after its plain command exited 0:
#  1. the JIT / parity / edge / sharded GPU tests;
#  2. the default bench line, its ncu launch list;
#  3. ncu --set full of one steady step of the kept schedule (forced by env $2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2fin2}; F=${2:-"SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=0"}; S=${3:-4}; C=${4:-4}
timeout 1200 python -m pytest tests/test_jit.py tests/test_gpu_parity.py tests/test_edge_gpu.py tests/test_sharded_gpu.py -m gpu -q --durations=8 > gpurun_out/${T}_tests_subset.log 2>&1; echo "subset rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_launch.log 2>&1
echo "bench+launch list rc=$?"
timeout 300 env $F python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 env $F ncu --set full --import-source on --clock-control none -k regex:sdb_pass -s $S -c $C -o gpurun_out/${T}_full \
  python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu-baseline --no-other-configs > gpurun_out/${T}_ncu_full.log 2>&1
echo "full rc=$?"
