cd /root/repo
for r in 4 5; do
  SDB_RBITS=$r timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5c_all_$r.log 2>&1
  SDB_RBITS=$r timeout 900 python bench.py --config 5 --n 28 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r5c_c5_$r.log 2>&1
done
