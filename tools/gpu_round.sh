#!/bin/bash
# One GPU session: parity tests, bench, reference arm, stage times, ncu launch
# list, ncu --set full of the hot kernels (summaries made on the box; the
# C4 reports are kept, the C3 ones are summarised and dropped to stay under
# the 64 MiB copy-back limit).  Outputs under gpurun_out/$TAG.
TAG=${TAG:-r1}
O=gpurun_out/$TAG
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>>$O/bench.err
cat $O/bench_ref.json
python tools/stage_times.py C3 --reps 10 > $O/stages_c3.txt 2>&1
python tools/stage_times.py C4 --reps 10 > $O/stages_c4.txt 2>&1
cat $O/stages_c3.txt $O/stages_c4.txt | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-extra > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
for C in C4 C3; do
ncu --set full --clock-control none --import-source on -k regex:"k_hist|k_plan|k_tma_pass|k_pass_bytes|k_vs" -c 7 \
  -o $O/full_sort_$C -f python tools/stage_times.py $C --reps 1 > $O/ncu_full_sort_$C.log 2>&1; echo "ncu sort $C rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_emit|k_table" -c 5 \
  -o $O/full_emit_$C -f python tools/stage_times.py $C --reps 1 > $O/ncu_full_emit_$C.log 2>&1; echo "ncu emit $C rc=$?"
python tools/ncu_summary.py full $O/full_sort_$C.ncu-rep > $O/${TAG}_${C}_sort_full.md
python tools/ncu_summary.py full $O/full_emit_$C.ncu-rep > $O/${TAG}_${C}_emit_full.md
python tools/traffic.py $C=$O/full_sort_$C.ncu-rep,$O/full_emit_$C.ncu-rep > $O/traffic_$C.json 2>&1
done
python tools/ncu_summary.py launches $O/launches_bench.csv > $O/${TAG}_launches.md
rm -f $O/full_sort_C3.ncu-rep $O/full_emit_C3.ncu-rep
du -sh $O
