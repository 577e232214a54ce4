#!/bin/bash
for C in C5 C1; do timeout 600 python tools/stage_times.py $C --reps 5 --check --no-flush 2>&1 | grep -E "n=|plan|sort|emit|table|total|digest|rror"; done
