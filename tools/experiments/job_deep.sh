# slow-case set: before (deep off, short off) / after (deep on, short 64 MB)
echo "== off"; TL_TTV_DEEP_MIN_K=0 TL_TTV_SHORT_MB=0 timeout 600 python tools/experiments/ttv_cases.py
echo "== on"; TL_TTV_SHORT_MB=64 timeout 600 python tools/experiments/ttv_cases.py
TL_TTV_SHORT_MB=64 timeout 900 python -m pytest tests -m gpu -q -x -k "ttv or parity or fuzz or views or l2keep" -p no:cacheprovider 2>&1 | tail -2
