#!/bin/bash
# sort stage time of variants (no digest: experiment builds may produce invalid output)
for v in "" $@; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  NDX_LIB=$lib timeout 200 python tools/stage_times.py C4 --reps 10 --no-flush --stages 2 2>&1 | grep -E "sort|rror"
done
