#!/bin/bash
# CZ -> CNOT conversion + look-ahead growth: parity tests, then A/B bench
# (new default vs SDB_CZ_CX=0 SDB_LOOKAHEAD=0), then the full default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2s5p}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_oracle_gpu.py tests/test_sharded_gpu.py -q -x --durations=10 > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
Q="--no-e2e --no-cpu-baseline --no-other-configs --steps 20 --warmup 5"
timeout 600 python bench.py $Q > gpurun_out/${T}_new.json 2> gpurun_out/${T}_new.err; echo "new rc=$?"
timeout 600 env SDB_CZ_CX=0 SDB_LOOKAHEAD=0 python bench.py $Q > gpurun_out/${T}_old.json 2> gpurun_out/${T}_old.err; echo "old rc=$?"
timeout 600 python bench.py $Q > gpurun_out/${T}_new2.json 2> gpurun_out/${T}_new2.err; echo "new2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
