#!/bin/bash
# One GPU session producing the round's evidence under gpurun_out/:
#   bench line, ncu launch list of the bench command, ncu --set full of the
#   ttv kernels (cfg2), the FP64 GETT (cfg3), the reductions, HOPM and cfg5.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
if [ -n "${PARITY_CFG3:-}" ]; then
TL_PARITY_REPORT=$PWD/gpurun_out/parity_report.jsonl timeout 1200 python -m pytest tests -m gpu -q -k cfg3_ttm_full_size \
    > gpurun_out/parity_cfg3.log 2>&1
fi
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
CMD="python bench.py --steps 2 --warmup 3 --no-components --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_ncu.log 2>&1
tools/ncu_box.sh prof_ttv "ttv_" cfg2
tools/ncu_box.sh prof_ttm "ttm_dmma" cfg3
tools/ncu_box.sh prof_red "dot_" cfg2
tools/ncu_box.sh prof_hopm "ttv_" cfg4
tools/ncu_box.sh prof_cfg5 "ttv_|ttm_|dot_" cfg5
tools/ncu_box.sh prof_copy "copy" copy
tools/ncu_box.sh prof_few "ttm_few" few
# every layout x every mode of the configs' shapes (profiles/config_sweep_<tag>.md via tools/summarize_sweep.py)
timeout 1200 python tools/experiments/config_sweep.py ttv2,ttv4,ttv5,ttm3,ttm5,inner 8 > gpurun_out/config_sweep.jsonl 2> gpurun_out/config_sweep.err
TL_TTM_FEW=0 timeout 600 python tools/experiments/config_sweep.py ttm5 8 > gpurun_out/config_sweep_ttm5_before.jsonl 2>> gpurun_out/config_sweep.err
tools/experiments/hopm_dram.sh
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
