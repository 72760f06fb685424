# stream ttm: K mod 4 tail as a zero-padded DMMA k-step (0) or per-lane FMAs (1); ncu cold + graph-replay times, sha
export NCU_EXTRA="--profile-from-start off"
for r in 1 2; do for d in 0 1; do
  TL_TTM_DFMA_TAIL=$d tools/ncu_times.sh dfma_$d "ttm_" python tools/experiments/ttm5_once.py | awk -v d=$d '{s+=$3; n++} END {printf "dfma=%s ncu cold mean %.2f us (%d)\n", d, s/n, n}'
  TL_TTM_DFMA_TAIL=$d TL_FUSED_NORM=0 tools/ncu_times.sh dfmap_$d "ttm_" python tools/experiments/ttm5_once.py | awk -v d=$d '{s+=$3; n++} END {printf "dfma=%s plain ncu cold mean %.2f us (%d)\n", d, s/n, n}'
  echo -n "dfma=$d "; TL_TTM_DFMA_TAIL=$d timeout 200 python tools/experiments/sweep_ttm5.py | tail -1
done; done
TL_TTM_DFMA_TAIL=1 timeout 600 python -m pytest tests -m gpu -q -x -k "stream or ttm" -p no:cacheprovider 2>&1 | tail -1
