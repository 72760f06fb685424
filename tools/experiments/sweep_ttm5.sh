set -u
for cfg in "2 1" "2 2" "3 1" "3 2" "4 1" "2 4"; do set -- $cfg
  echo "st=$1 nt=$2 $(TL_TTM_BULK_ST=$1 TL_TTM_BULK_NT=$2 timeout 120 python tools/experiments/sweep_ttm5.py 2>&1 | tail -1)"
done
