#!/bin/bash
O=gpurun_out/r2i
mkdir -p $O
for C in C4 C3 C1; do timeout 300 python tools/stage_times.py $C --reps 10 --check 2>&1 | grep -E "sort|total|digest|rror"; done > $O/t.txt 2>&1; cat $O/t.txt
timeout 300 python tools/stage_times.py C5 --reps 5 2>&1 | grep -E "sort|total|rror"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
