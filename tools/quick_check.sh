#!/bin/bash
O=gpurun_out/r2p
mkdir -p $O
for C in C4 C3; do timeout 300 python tools/stage_times.py $C --reps 10 --check --no-flush 2>&1 | grep -E "plan|sort|emit|total|digest|rror"; done
timeout 900 python -m pytest tests/test_wah_gpu.py -x -q 2>&1 | tail -2
