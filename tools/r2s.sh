#!/bin/bash
# pass B / wide pass writing rows only (experiment: output not valid for the emit)
for v in "" rows; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  for C in C4 C3; do NDX_LIB=$lib timeout 200 python tools/stage_times.py $C --reps 10 --no-flush 2>&1 | grep -E "sort|rror"; done
done
