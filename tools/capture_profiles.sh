#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU): launch list of the default
# bench command and one `ncu --set full` capture of the tile-pass kernels of a
# config-4 n=30 step (passes 0..3: WHT-only, CZ, WHT-only, diagonal table).
cd "$(dirname "$0")/.."
TAG=${1:-r1}
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cap_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cap_ncu_launch.log 2>&1
timeout 300 python tools/profile_pass.py 4 30 1 > gpurun_out/cap_pp.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sdb_pass|k_tile_pass" -s 0 -c 4 \
  -o gpurun_out/${TAG}_full python tools/profile_pass.py 4 30 1 > gpurun_out/cap_ncu_full.log 2>&1
