#!/bin/bash
# full ncu capture of the rows-form helper kernels (k_vs, k_tile_heads) on C4
O=gpurun_out/r2v; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vs|k_tile_heads" -c 2 -o $O/helpers -f python tools/stage_times.py C4 --reps 1 --no-flush > $O/ncu.log 2>&1
tail -3 $O/ncu.log
