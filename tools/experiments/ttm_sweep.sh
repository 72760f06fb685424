for cfg in "28 4" "28 8" "16 4" "40 4" "56 8" "20 8"; do set -- $cfg; echo "== stage ${1}KB NT $2"; TL_TTM_STAGE_KB=$1 TL_TTM_NT=$2 timeout 120 python tools/experiments/probe_ops.py cfg5 2>&1 | grep ttm; done
echo "== SIMT 28"; TL_TTM_SIMT=1 TL_TTM_STAGE_KB=28 timeout 120 python tools/experiments/probe_ops.py cfg5 2>&1 | grep ttm
echo "== SIMT 12"; TL_TTM_SIMT=1 TL_TTM_STAGE_KB=12 timeout 120 python tools/experiments/probe_ops.py cfg5 2>&1 | grep ttm
