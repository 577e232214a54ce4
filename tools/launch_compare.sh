#!/bin/bash
# per-kernel launch list of the C4 build: product vs base build
O=gpurun_out/launch_compare; mkdir -p $O
for v in "" base; do
  lib=libndx.so; [ -n "$v" ] && lib=libndx_$v.so
  NDX_LIB=$lib timeout 200 python tools/stage_times.py C4 --reps 10 --no-flush 2>&1 | grep -E "sort|emit|total"
  NDX_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$v.csv python tools/stage_times.py C4 --reps 1 --no-flush > /dev/null 2>&1
done
