#!/bin/bash
O=gpurun_out/r2j
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -5 $O/bench.err
python tools/stage_times.py C4 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tma_pass|k_emit|k_hist" -s 4 -c 6 \
  -o $O/full_C4 -f python tools/stage_times.py C4 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py full $O/full_C4.ncu-rep > $O/full_C4.md
cat $O/full_C4.md
