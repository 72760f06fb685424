#!/bin/bash
# HOPM cfg4 sweeps/s with and without the early-prefetch PDL between small folds
for e in 0 1 0 1; do echo -n "early=$e: "; TL_HOPM_EARLY=$e python tools/experiments/hopm_rate.py; done
