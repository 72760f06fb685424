# ncu --set full with source of the cfg5 stream ttm, cold (cache flush) and L2-warm (no flush), plain and fused
mkdir -p gpurun_out
for fn in 0 1; do for cc in all none; do
  TL_FUSED_NORM=$fn timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control $cc \
     -k regex:ttm_stream -c 2 -o gpurun_out/t5_${fn}_${cc} python tools/experiments/ttm5_once.py > gpurun_out/t5_${fn}_${cc}.log 2>&1
  ncu -i gpurun_out/t5_${fn}_${cc}.ncu-rep --page source --csv --print-source sass > gpurun_out/t5_${fn}_${cc}_src.csv 2>/dev/null; gzip -f gpurun_out/t5_${fn}_${cc}_src.csv
  ncu -i gpurun_out/t5_${fn}_${cc}.ncu-rep --page details --csv > gpurun_out/t5_${fn}_${cc}_det.csv 2>/dev/null; gzip -f gpurun_out/t5_${fn}_${cc}_det.csv
  rm -f gpurun_out/t5_${fn}_${cc}.ncu-rep
done; done
ls -la gpurun_out/t5_*
