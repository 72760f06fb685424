# A/B: HEAD stream ttm (A) vs reduced k-step unroll for the two-m16-tile instantiations (B)
for r in 1 2 3; do for v in A B; do echo -n "$v: "; TL_LIB=abl/lib$v.so timeout 200 python tools/experiments/sweep_ttm5.py | tail -1; done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "stream or ttm" -p no:cacheprovider 2>&1 | tail -1
