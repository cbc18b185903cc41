# A/B: pre_keep = prelude graph; step = plus one fused scale/check/next kernel in the graph body
set -x
for r in 1 2; do
for v in pre_keep step; do
  for c in C2 C3 C4 C5; do HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py $c 11; done
done
done
