#!/bin/bash
# HOPM cfg4: MB of A kept L2-resident between the two passes (0 = off)
for mb in ${MBS:-0 32 64 96 0 32 64 96}; do TL_HOPM_KEEP_MB=$mb timeout 200 python tools/experiments/hopm_keep.py; done
