#!/bin/bash
# per-kernel launch list + full ncu of the compact passes (C4)
O=gpurun_out/r2b
mkdir -p $O
python tools/stage_times.py C4 --reps 2 > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python tools/stage_times.py C4 --reps 1 > $O/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/stage_times.py C3 --reps 2 > $O/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python tools/stage_times.py C3 --reps 1 > $O/ncu_launch3.log 2>&1; echo "ncu launch3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass" -s 2 -c 2 \
  -o $O/full_ab_C4 -f python tools/stage_times.py C4 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py launches $O/launches_c4.csv > $O/launches_c4.md
python tools/ncu_summary.py launches $O/launches_c3.csv > $O/launches_c3.md
python tools/ncu_summary.py full $O/full_ab_C4.ncu-rep > $O/full_ab_C4.md
cat $O/launches_c4.md $O/launches_c3.md $O/full_ab_C4.md
