# A/B of environment switches on one library build: interleaved C-config solves (scripts/ab_time.py),
#   bash scripts/ab_env.sh C5 "HD_LSA_REV=0" "HD_STENCIL_TMA=0" ...   (each argument: one variant's env; "" = defaults)
cfg=$1; shift
for round in 1 2; do
  for v in "" "$@"; do
    echo "== [$v] round $round"
    env $v python scripts/ab_time.py $cfg 7 2>&1 | tail -1
  done
done
