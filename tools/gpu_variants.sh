#!/bin/bash
# Config-4 bench under several env variants (each "name:ENV=.. ENV2=.."),
# forced schedules bypass the autotuner. Usage: gpu_variants.sh TAG "a:X=1" "b:X=2 Y=3" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=$1; shift
Q="--no-e2e --no-cpu-baseline --no-other-configs --steps 20 --warmup 5"
for v in "$@"; do
  name=${v%%:*}; envs=${v#*:}
  timeout 900 env $envs python bench.py $Q > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  echo "$name rc=$?"
done
