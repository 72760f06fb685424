#!/bin/bash
# cold (ncu) duration of the cfg5 stream ttm over consumer warps x tile target x output tiles per warp
export NCU_EXTRA="--profile-from-start off"
for ob in ${OBS:-2}; do for nw in ${NWS:-4 6 8}; do for kb in ${KBS:-6 8 12 16}; do
  TL_TTM_STREAM_OB=$ob TL_TTM_STREAM_NW=$nw TL_TTM_STREAM_KB=$kb tools/ncu_times.sh s_${ob}_${nw}_${kb} "ttm_" python tools/experiments/ttm5_once.py \
    | awk -v nw=$nw -v kb=$kb -v ob=$ob '{s+=$3; n++} END {printf "ob=%s nw=%s kb=%s mean %.2f us (%d)\n", ob, nw, kb, s/n, n}'
done; done; done
