#!/bin/bash
# Whole-group configs 3 and 5 (n=28): register coordinates x ring pipeline.
cd "$(dirname "$0")/.."
for e in "SDB_RBITS=4 SDB_RING=1" "SDB_RBITS=5 SDB_RING=1"; do
  tag=$(echo $e | tr -d ' =')
  env SDB_SPLIT_DIAG=0 $e timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/c35_3_$tag.log 2>&1
  env SDB_SPLIT_DIAG=0 $e timeout 900 python bench.py --config 5 --n 28 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/c35_5_$tag.log 2>&1
done
env SDB_SPLIT_DIAG=0 SDB_RING=0 timeout 900 python bench.py --config 5 --n 28 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/c35_5_ring0.log 2>&1
