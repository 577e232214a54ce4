for v in ${VARS:-v0 v1 v2 v3 v4}; do
  echo "== $v"
  NDX_LIB=libndx_$v.so python tools/stage_times.py C3 --reps 10 2>&1 | grep -E "sort|emit"
  NDX_LIB=libndx_$v.so python tools/stage_times.py C4 --reps 10 --check 2>&1 | grep -E "sort|emit|digest"
done
