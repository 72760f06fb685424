# mixed-layout inner: HEAD kernel vs the pipelined float kernel at 2 / 3 / 4 CTAs per SM of registers
for r in 1 2; do for v in H 2 3 4; do echo -n "$v: "; TL_LIB=abl/lib$v.so timeout 200 python tools/experiments/inner_mixed.py; done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "inner or norm or reduce" -p no:cacheprovider 2>&1 | tail -1
