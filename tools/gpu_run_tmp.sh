for v in "h1:SDB_DRAM_PATTERN=1" "h0:SDB_DRAM_PATTERN=0" "h1pf0:SDB_DRAM_PATTERN=1 SDB_PREFETCH=0" "h0pf0:SDB_DRAM_PATTERN=0 SDB_PREFETCH=0"; do
  lab=${v%%:*}; ev=${v#*:}
  env $ev timeout 300 python tools/profile_pass.py 4 30 1 > gpurun_out/pp_$lab.log 2>&1
  env $ev timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sdb_pass --csv --log-file gpurun_out/launches_$lab.csv python tools/profile_pass.py 4 30 1 > /dev/null 2>&1
  echo "$lab"; python - "$lab" <<'PY'
import csv,sys
lab=sys.argv[1]
rows=[r for r in csv.reader(open(f'gpurun_out/launches_{lab}.csv')) if len(r)>10 and r[0]!='ID']
t=[round(float(r[-1])/1e6,2) for r in rows]; print(t, round(sum(t),2))
PY
done
