#!/bin/bash
# plan stage time of variants (no digest: experiment builds may produce invalid output)
for v in "" $@; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  for C in C4 C3; do NDX_LIB=$lib timeout 200 python tools/stage_times.py $C --reps 10 --no-flush --stages 1 2>&1 | grep -E "plan|rror"; done
done
