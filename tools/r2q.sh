#!/bin/bash
for v in "" l8alias base_alias; do
  echo "== $v"
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  NDX_LIB=$lib timeout 200 python tools/stage_times.py C4 --reps 10 --check --no-flush 2>&1 | grep -E "sort|digest|rror"
done
