# GETT: one CTA per tile vs persistent CTAs with cross-tile prefetch (TL_GETT_PERSIST CTAs per SM)
for p in 0 2 3 0 2 3; do echo -n "persist=$p "; TL_GETT_PERSIST=$p timeout 300 python tools/experiments/cfg3_tile.py; done
for p in 0 3; do TL_GETT_PERSIST=$p timeout 900 python -m pytest tests -m gpu -q -x -k "ttm or gett or ttt or fuzz" -p no:cacheprovider 2>&1 | tail -1; done
