# cfg5 stream ttm (ncu, cold): CTAs per SM x consumer warps, plain and fused norm; then the GPU ttm tests on the best
mkdir -p gpurun_out
export NCU_EXTRA="--profile-from-start off"
for fn in 0 1; do for cfg in "1 8" "2 4" "2 5" "2 6" "3 3" "3 4"; do set -- $cfg
  TL_FUSED_NORM=$fn TL_TTM_STREAM_CPS=$1 TL_TTM_STREAM_NW=$2 tools/ncu_times.sh cps_${fn}_$1_$2 "ttm_" python tools/experiments/ttm5_once.py \
    | awk -v fn=$fn -v c=$1 -v w=$2 '{s+=$3; n++; k=$NF} END {printf "fused=%s cps=%s nw=%s mean %.2f us (%d) %s\n", fn, c, w, s/n, n, k}'
done; done 2>&1 | tee gpurun_out/cps.txt
for cfg in "2 4" "2 6"; do set -- $cfg; TL_TTM_STREAM_CPS=$1 TL_TTM_STREAM_NW=$2 timeout 300 python -m pytest tests -m gpu -q -x -k "stream or ttm" -p no:cacheprovider 2>&1 | tail -1; done
