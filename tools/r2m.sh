#!/bin/bash
O=gpurun_out/r2m
mkdir -p $O
for C in C4 C3; do timeout 300 python tools/stage_times.py $C --reps 10 --check 2>&1 | grep -E "plan|sort|emit|total|digest|rror"; done > $O/t.txt 2>&1; cat $O/t.txt
timeout 900 python -m pytest tests/test_wah_gpu.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
