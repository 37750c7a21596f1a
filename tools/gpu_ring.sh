#!/bin/bash
# Ring-pipeline check: JIT parity (small n, also with few CTAs so each runs
# many tiles), full-size oracle parity, then bench A/B against the two-CTA kernel.
cd "$(dirname "$0")/.."
O=gpurun_out
SDB_RING=1 timeout 600 python -m pytest tests/test_jit.py -m gpu -x -q > $O/ring_jit.log 2>&1; echo "rc=$?" >> $O/ring_jit.log
SDB_RING=1 SDB_MAX_CTAS=3 timeout 600 python -m pytest tests/test_jit.py -m gpu -x -q > $O/ring_jit3.log 2>&1; echo "rc=$?" >> $O/ring_jit3.log
for r in 1 0 1; do
  SDB_RING=$r timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-other-configs > $O/ring_bench_$r.log 2>&1; echo "rc=$?" >> $O/ring_bench_$r.log
  mv $O/ring_bench_$r.log $O/ring_bench_${r}_$(date +%s).log
done
SDB_RING=1 timeout 900 python -m pytest tests/test_fullsize_oracle_gpu.py -m gpu -x -q > $O/ring_full.log 2>&1; echo "rc=$?" >> $O/ring_full.log
