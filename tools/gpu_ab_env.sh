#!/bin/bash
# A/B of the default bench (config 4) against the same bench under env "$2"
# (e.g. "SDB_CX_BATCH=0"), interleaved new/old/new, then optional tests "$3".
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-ab}; OLD=${2:-SDB_NOP=1}; TESTS=${3:-}
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -q -x --durations=10 > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"
fi
Q="--no-e2e --no-cpu-baseline --no-other-configs --steps 20 --warmup 5"
timeout 600 python bench.py $Q > gpurun_out/${T}_new.json 2> gpurun_out/${T}_new.err; echo "new rc=$?"
timeout 600 env $OLD python bench.py $Q > gpurun_out/${T}_old.json 2> gpurun_out/${T}_old.err; echo "old rc=$?"
timeout 600 python bench.py $Q > gpurun_out/${T}_new2.json 2> gpurun_out/${T}_new2.err; echo "new2 rc=$?"
