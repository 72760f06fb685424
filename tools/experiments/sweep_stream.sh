# config-5 ttm: stream kernel (default) vs the bulk kernel (kb=0)
set -u
for kb in 0 12 12; do
  echo "kb=$kb $(TL_TTM_STREAM_KB=$kb timeout 60 python tools/experiments/sweep_ttm5.py 2>&1 | tail -1)"
done
