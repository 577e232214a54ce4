#!/bin/bash
O=gpurun_out/r2d
mkdir -p $O
for mode in 0 1; do for lib in libndx.so libndx_nocarve.so; do
echo "== host_dispatch=$mode lib=$lib"
NDX_HOST_DISPATCH=$mode NDX_LIB=$lib python tools/stage_times.py C4 --reps 10 2>&1 | grep -E "sort|total"
NDX_HOST_DISPATCH=$mode NDX_LIB=$lib python tools/stage_times.py C3 --reps 10 2>&1 | grep -E "sort|total"
done; done > $O/cdp.txt 2>&1
cat $O/cdp.txt
