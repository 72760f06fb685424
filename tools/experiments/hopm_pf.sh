#!/bin/bash
# HOPM cfg4 sweeps/s vs the L2 warm-up budget (side-stream prefetch branch).
for mb in 0 48 96 128; do
  echo -n "prefetch ${mb} MB: "; TL_HOPM_PREFETCH_MB=$mb python tools/experiments/hopm_rate.py
  echo -n "prefetch ${mb} MB, no join: "; TL_HOPM_PF_NOJOIN=1 TL_HOPM_PREFETCH_MB=$mb python tools/experiments/hopm_rate.py
done
