#!/bin/bash
# Ring pipeline (with TMA stores) forced on/off for the whole-group configs 2 and 3.
cd "$(dirname "$0")/.."
for c in 3 2; do
  for r in 0 1; do
    SDB_RING=$r timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/cr_${c}_${r}.log 2>&1
  done
done
