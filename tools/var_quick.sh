# Quick A/B of libndx variants on C4 and C3 (tools/variants.py builds them):
#   VARS="vb" bash tools/var_quick.sh
for v in base ${VARS} base ${VARS}; do
  if [ "$v" = base ]; then L=libndx.so; else L=libndx_$v.so; fi
  echo "== $v"
  NDX_LIB=$L python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|emit|total|digest"
  NDX_LIB=$L python tools/stage_times.py C3 --reps 10 2>&1 | grep -E "sort|total"
done
