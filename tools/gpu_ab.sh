#!/bin/bash
# A/B per-pass launch times of one config-4 n=30 step under env settings: gpu_ab.sh "ENV=1" "ENV=0" ...
cd "$(dirname "$0")/.."
i=0
for e in "$@"; do
  env $e timeout 300 python tools/profile_pass.py 4 30 1 > gpurun_out/ab_plain_$i.log 2>&1 && \
  env $e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sdb_pass|k_tile_pass" --csv --log-file gpurun_out/ab_$i.csv python tools/profile_pass.py 4 30 1 > gpurun_out/ab_ncu_$i.log 2>&1
  echo "$e" > gpurun_out/ab_$i.env
  i=$((i+1))
done
