#!/bin/bash
# One GPU round trip: GPU tests, a short bench, per-pass launch times of one
# config-4 step at n=30 (ncu launch list).
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_pass.py ${CFG:-4} ${N:-30} 1 > gpurun_out/pp30.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tile_pass --csv --log-file gpurun_out/launches_pp30.csv python tools/profile_pass.py ${CFG:-4} ${N:-30} 1 > gpurun_out/ncu_l.log 2>&1
