#!/bin/bash
# full ncu capture of pass A and pass B (C4) and k_hist
O=gpurun_out/r2aa; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass|k_hist" --launch-skip 0 --launch-count 4 -o $O/passes -f python tools/stage_times.py C4 --reps 1 --no-flush > $O/ncu.log 2>&1
tail -2 $O/ncu.log
