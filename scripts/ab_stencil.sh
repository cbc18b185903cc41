set -x
for r in 1 2; do
for v in base minb4 ring2 ring2minb4; do
  HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py C5 7
  HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py C3 15
done
done
