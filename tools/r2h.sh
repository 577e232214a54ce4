#!/bin/bash
O=gpurun_out/r2h
mkdir -p $O
for v in "" balias aalias both walias; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  NDX_LIB=$lib timeout 200 python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|digest|rror"
  NDX_LIB=$lib timeout 200 python tools/stage_times.py C3 --reps 10 --check 2>&1 | grep -E "sort|digest|rror"
done > $O/variants.txt 2>&1
cat $O/variants.txt
