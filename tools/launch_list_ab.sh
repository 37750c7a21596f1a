#!/bin/bash
# Per-launch times (ncu launch list, cold/serialised) of one config-4 step with
# the per-term schedule forced, for each env setting: tools/launch_list_ab.sh TAG "ENV" ...
cd "$(dirname "$0")/.."
tag=$1; shift
i=0
for e in "$@"; do
  env SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=2 $e timeout 300 python tools/profile_pass.py 4 30 2 > gpurun_out/ll_${tag}_${i}.log 2>&1 && \
  env SDB_SPLIT_DIAG=1 SDB_MAX_HDEPTH=2 $e timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sdb_pass --csv \
    --log-file gpurun_out/ll_${tag}_${i}.csv python tools/profile_pass.py 4 30 2 > gpurun_out/ll_${tag}_${i}_ncu.log 2>&1
  echo "$e" > gpurun_out/ll_${tag}_${i}.env
  i=$((i+1))
done
