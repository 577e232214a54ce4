#!/bin/bash
O=gpurun_out/r2e
mkdir -p $O
python tools/stage_times.py C4 --reps 10 --check > $O/c4.txt 2>&1; cat $O/c4.txt
python tools/stage_times.py C3 --reps 10 --check > $O/c3.txt 2>&1; cat $O/c3.txt
for v in lb2 lb0 bmin3 bc; do
  echo "== $v"
  NDX_LIB=libndx_$v.so timeout 200 python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|digest|rror"
done > $O/variants.txt 2>&1
cat $O/variants.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python tools/stage_times.py C4 --reps 1 > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass" -s 6 -c 3 \
  -o $O/full_ab_C4 -f python tools/stage_times.py C4 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py launches $O/launches_c4.csv > $O/launches_c4.md
python tools/ncu_summary.py full $O/full_ab_C4.ncu-rep > $O/full_ab_C4.md
cat $O/launches_c4.md $O/full_ab_C4.md
