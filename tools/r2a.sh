#!/bin/bash
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
for C in C4 C3 C1; do timeout 300 python tools/stage_times.py $C --reps 10 --check > $O/stages_$C.txt 2>&1; echo "rc=$?" >> $O/stages_$C.txt; done
cat $O/stages_C4.txt $O/stages_C3.txt $O/stages_C1.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
for v in v1 v2 v3 v4; do
  echo "== $v"
  NDX_LIB=libndx_$v.so timeout 200 python tools/stage_times.py C3 --reps 10 --check 2>&1 | grep -E "sort|emit|digest|rror"
  NDX_LIB=libndx_$v.so timeout 200 python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|emit|digest|rror"
done > $O/variants.txt 2>&1
cat $O/variants.txt
