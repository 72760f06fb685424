set -u
for cfg in "2 2 14" "2 2 28" "2 2 40" "3 2 28" "2 1 28"; do set -- $cfg
  echo "st=$1 nt=$2 kb=$3 $(TL_TTM_BULK_ST=$1 TL_TTM_BULK_NT=$2 TL_TTM_BULK_KB=$3 timeout 120 python tools/experiments/sweep_ttm5.py 2>&1 | tail -1)"
done
