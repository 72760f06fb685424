set -u
for cfg in "3 10" "3 14" "4 14" "3 20" "4 20" "3 28"; do set -- $cfg
  echo "st=$1 kb=$2 $(TL_TTM_BULK_ST=$1 TL_TTM_BULK_KB=$2 timeout 120 python tools/scratch/sweep_ttm5.py 2>&1 | tail -1)"
done
