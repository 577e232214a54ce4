#!/bin/bash
# sharded step at N=1, C5 and C1 stage times
O=gpurun_out/r2cc; mkdir -p $O
timeout 600 python bench.py --force-sharded --steps 10 --warmup 3 > $O/sharded_n1.json 2> $O/sharded_n1.err; echo "sharded rc=$?"
tail -c 1500 $O/sharded_n1.json
timeout 600 python tools/stage_times.py C5 --reps 5 --check --no-flush > $O/stages_c5.txt 2>&1; cat $O/stages_c5.txt
timeout 300 python tools/stage_times.py C1 --reps 10 --check --no-flush > $O/stages_c1.txt 2>&1; cat $O/stages_c1.txt
