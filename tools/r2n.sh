#!/bin/bash
O=gpurun_out/r2n
mkdir -p $O
timeout 600 python bench.py --force-sharded --steps 10 --warmup 3 --e2e-steps 2 > $O/fs.json 2>$O/fs.err; echo rc=$?
python -c "import json;d=json.load(open('$O/fs.json'));print(d['ms_per_step'], d['gather_to_rank0_ms'], d['result_check'])"
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q -k "device_counts or dist_build" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --force-sharded --steps 2 --warmup 3 --e2e-steps 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'P'
import csv,collections
rows=list(csv.reader(open('gpurun_out/r2n/launches.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.OrderedDict()
for r in rows[start+1:]:
    if len(r)>vi:
        k=r[ki][:50]; agg.setdefault(k,[]).append(float(r[vi]))
for k,v in agg.items(): print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v)/1000:9.1f} us")
P
