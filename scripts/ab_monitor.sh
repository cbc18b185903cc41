# A/B of the graph body's monitor placement (HD_MON_SIDE=1: side branch, lagged check; 0: main chain)
set -x
for r in 1 2; do
for m in 0 1; do
  for c in C5 C3 C4 C2; do HD_MON_SIDE=$m timeout 300 python scripts/ab_time.py $c 9; done
done
done
