#!/bin/bash
# rows-form stream: stage times + parity
for C in C4 C3; do timeout 300 python tools/stage_times.py $C --reps 10 --check --no-flush 2>&1 | grep -E "plan|sort|emit|table|total|digest|rror"; done
timeout 900 python -m pytest tests/test_wah_gpu.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q 2>&1 | tail -5
