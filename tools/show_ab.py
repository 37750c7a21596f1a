import csv, glob, os
for f in sorted(glob.glob('gpurun_out/ab_*.csv')):
    i = f.split('_')[-1].split('.')[0]
    env = open(f'gpurun_out/ab_{i}.env').read().strip()
    rows = [r for r in csv.DictReader([l for l in open(f) if l.startswith('"')])]
    v = [float(r['Metric Value']) / 1e6 for r in rows]
    print(env, [round(x, 2) for x in v], 'sum', round(sum(v), 2))
