#!/bin/bash
# HOPM cfg4 sweeps/s with and without the tail fold (mode-3 chain)
for tf in 0 1 0 1; do echo -n "tailfold=$tf: "; TL_HOPM_TAILFOLD=$tf python tools/experiments/hopm_rate.py; done
