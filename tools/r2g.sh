#!/bin/bash
O=gpurun_out/r2g
mkdir -p $O
for lib in libndx.so libndx_early.so; do
echo "== $lib"
NDX_LIB=$lib python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|total|digest"
NDX_LIB=$lib python tools/stage_times.py C3 --reps 10 --check 2>&1 | grep -E "sort|total|digest"
NDX_LIB=$lib python tools/stage_times.py C5 --reps 5 2>&1 | grep -E "sort|total|digest"
done > $O/t.txt 2>&1; cat $O/t.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python tools/stage_times.py C4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass" -s 6 -c 3 \
  -o $O/full_ab_C4 -f python tools/stage_times.py C4 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py full $O/full_ab_C4.ncu-rep > $O/full_ab_C4.md
cat $O/full_ab_C4.md
