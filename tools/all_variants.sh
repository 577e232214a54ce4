#!/bin/bash
# whole-build variants (NDX_LIB) on C4 and C3: every stage, digests
for v in "" $@; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  for C in C4 C3; do NDX_LIB=$lib timeout 200 python tools/stage_times.py $C --reps 10 --check --no-flush 2>&1 | grep -E "plan|sort|emit|total|digest|rror"; done
done
