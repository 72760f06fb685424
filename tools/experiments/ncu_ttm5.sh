set -u
mkdir -p gpurun_out
for kb in 0 14; do
TL_TTM_BULK_KB=$kb TL_TTM_BULK_NT=2 timeout 120 python tools/experiments/ncu_ttm5.py || exit 1
TL_TTM_BULK_KB=$kb TL_TTM_BULK_NT=2 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ttm_ -o gpurun_out/ttm5_$kb python tools/experiments/ncu_ttm5.py > gpurun_out/ttm5_$kb.log 2>&1
ncu -i gpurun_out/ttm5_$kb.ncu-rep --page details --csv > gpurun_out/ttm5_${kb}_details.csv
ncu -i gpurun_out/ttm5_$kb.ncu-rep --page source --csv > gpurun_out/ttm5_${kb}_source.csv; gzip -f gpurun_out/ttm5_${kb}_source.csv
rm -f gpurun_out/ttm5_$kb.ncu-rep
done
