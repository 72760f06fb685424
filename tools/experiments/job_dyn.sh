# cfg5 stream ttm (ncu cold): static vs dynamic tile hand-out, plain and fused
mkdir -p gpurun_out
export NCU_EXTRA="--profile-from-start off"
for r in 1 2; do for fn in 0 1; do for dyn in 0 1; do
  TL_FUSED_NORM=$fn TL_TTM_STREAM_DYN=$dyn tools/ncu_times.sh dyn_${fn}_${dyn} "ttm_" python tools/experiments/ttm5_once.py \
    | awk -v fn=$fn -v d=$dyn '{s+=$3; n++} END {printf "fused=%s dyn=%s mean %.2f us (%d)\n", fn, d, s/n, n}'
done; done; done 2>&1 | tee gpurun_out/dyn.txt
TL_TTM_STREAM_DYN=1 timeout 300 python -m pytest tests -m gpu -q -x -k "stream or ttm" -p no:cacheprovider 2>&1 | tail -1
