#!/bin/bash
O=gpurun_out/r2l
mkdir -p $O
python tools/stage_times.py C4 --reps 10 --no-flush 2>&1 | grep -E "plan|sort|emit|total"
python tools/stage_times.py C4 --reps 10 2>&1 | grep -E "plan|sort|emit|total"
python tools/stage_times.py C4 --reps 2 --no-flush > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python tools/stage_times.py C4 --reps 2 --no-flush > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/r2l/launches.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[start+1:]:
    if len(r)>vi: print(r[ki][:40], r[vi])
P
