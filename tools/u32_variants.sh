#!/bin/bash
# general keys (pairs form): stage times and digests of variants
for v in "" $@; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  NDX_LIB=$lib timeout 300 python tools/stage_times.py U32 --n 16777216 --reps 5 --check --no-flush 2>&1 | grep -E "plan|sort|emit|total|digest|rror"
done
