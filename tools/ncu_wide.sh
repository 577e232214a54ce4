#!/bin/bash
# full ncu capture of the wide pass on C3
O=gpurun_out/ncu_wide; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass" -c 1 -o $O/wide -f python tools/stage_times.py C3 --reps 1 --no-flush > $O/ncu.log 2>&1
tail -2 $O/ncu.log
