#!/bin/bash
# full ncu capture of k_emit_rows on C4
O=gpurun_out/r2x; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_emit_rows" -c 1 -o $O/emit_rows -f python tools/stage_times.py C4 --reps 1 --no-flush > $O/ncu.log 2>&1
tail -2 $O/ncu.log
