#!/bin/bash
# full GPU suite + stage times
for C in C4 C3; do timeout 300 python tools/stage_times.py $C --reps 10 --check --no-flush 2>&1 | grep -E "plan|sort|emit|total|digest|rror"; done
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5
