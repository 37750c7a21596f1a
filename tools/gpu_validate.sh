#!/bin/bash
# Validation of the current tree on one B200 (run under gpurun): smoke(), the
# full -m gpu suite, then the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2s5}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${T}_gputests.log 2>&1
echo "gpu tests rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
