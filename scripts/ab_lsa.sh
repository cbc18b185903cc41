# A/B of Arnoldi pass 1 item splits (HD_LSA_SPLIT builds, scripts/build_variant.sh)
set -x
for r in 1 2; do
for v in base split2 split4; do
  HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py C5 9
  HD_LIBRARY=_ab/libhelmdef_$v.so timeout 300 python scripts/ab_time.py C3 15
done
done
