#!/bin/bash
# Macro steps + split POINT stages: targeted parity tests, then config-4 bench variants.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2s5m}
timeout 1200 python -m pytest tests/test_edge_gpu.py tests/test_jit.py tests/test_gpu_parity.py -q -x \
  -k "macro or deep or cz_to_cnot or autotune" --durations=10 > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
bash tools/gpu_variants.sh $T "def:SDB_NOP=1" "nomacro:SDB_MACRO=0" "hd0split:SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=0" "macro3:SDB_MACRO=3"
