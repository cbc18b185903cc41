# A/B of the pre-loop: sync1 = one host synchronisation, eager launches; pre = the same captured as a cached graph
set -x
for r in 1 2; do
for v in sync1 pre; do
  for c in C2 C3 C4 C5; do HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py $c 11; done
done
done
