#!/bin/bash
O=gpurun_out/r2f
mkdir -p $O
python tools/stage_times.py C4 --reps 10 --check > $O/c4.txt 2>&1; cat $O/c4.txt
for v in w8 w2 amin2 bc; do
  echo "== $v"
  NDX_LIB=libndx_$v.so timeout 200 python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|digest|rror"
done > $O/variants.txt 2>&1
cat $O/variants.txt
python tools/stage_times.py C4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass" -s 6 -c 3 \
  -o $O/full_ab_C4 -f python tools/stage_times.py C4 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py full $O/full_ab_C4.ncu-rep > $O/full_ab_C4.md
cat $O/full_ab_C4.md
