#!/bin/bash
# A/B of env settings on the config-4 bench (alternating, twice each):
#   tools/gpu_ab_bench.sh TAG "ENV_A=.." "ENV_B=.."   (use "X=0" for the default)
cd "$(dirname "$0")/.."
tag=$1; shift
for rep in 1 2; do
  i=0
  for e in "$@"; do
    env $e timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/ab_${tag}_${i}_${rep}.log 2>&1
    echo "$e" >> gpurun_out/ab_${tag}_${i}_${rep}.log
    i=$((i+1))
  done
done
