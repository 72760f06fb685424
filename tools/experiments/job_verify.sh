mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log; tail -2 gpurun_out/gputest.log
for mb in 64 0; do TL_HOPM_KEEP_MB=$mb timeout 200 python tools/experiments/hopm_keep.py; done
export NCU_EXTRA="--profile-from-start off"
tools/ncu_times.sh ssq_fused "ttm_" python tools/experiments/ttm5_once.py | awk '{s+=$3; n++} END {printf "fused mean %.2f us (%d)\n", s/n, n}'
TL_FUSED_NORM=0 tools/ncu_times.sh ssq_plain "ttm_" python tools/experiments/ttm5_once.py | awk '{s+=$3; n++} END {printf "plain mean %.2f us (%d)\n", s/n, n}'
