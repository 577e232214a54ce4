#!/bin/bash
O=gpurun_out/r2k
mkdir -p $O
python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-extra > $O/plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-extra > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/ncu_summary.py launches $O/launches.csv > $O/launches.md; cat $O/launches.md
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/r2k/launches.csv')))
h=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[(r[ki][:40], r[vi]) for r in rows[start+1:] if len(r)>vi]
for k,v in seq[:60]: print(k, v)
P
