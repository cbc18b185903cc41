# A/B of programmatic graph edges (HD_PDL=1) on the final graph body
set -x
for r in 1 2; do
for m in 0 1; do
  for c in C2 C3 C4 C5; do HD_PDL=$m timeout 300 python scripts/ab_time.py $c 11; done
done
done
