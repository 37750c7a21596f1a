#!/bin/bash
cd "$(dirname "$0")/.."
tail -2 gpurun_out/pytest_gpu.log
grep metric gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],2), 'GB/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'step_frac', round(d['roofline']['step_frac'],3), 'norm_err', d['norm_error'])"
python -c "
import csv
rows=[r for r in csv.DictReader([l for l in open('gpurun_out/launches_pp30.csv') if l.startswith('\"')])]
v=[float(r['Metric Value'])/1e6 for r in rows]
print('per-pass ms', [round(x,2) for x in v], 'sum', round(sum(v),2))"
