# A/B of the pre-loop host synchronisations (base: three, sync1: one)
set -x
for r in 1 2; do
for v in base sync1; do
  for c in C2 C3 C4 C5; do HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py $c 11; done
done
done
