set -u
timeout 300 ncu --profile-from-start off --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:ttv_small -o gpurun_out/fold python tools/experiments/ncu_fold.py > gpurun_out/fold_ncu.log 2>&1
ncu -i gpurun_out/fold.ncu-rep --page source --csv > gpurun_out/fold_source.csv; gzip -f gpurun_out/fold_source.csv
ncu -i gpurun_out/fold.ncu-rep --page details --csv > gpurun_out/fold_details.csv
rm -f gpurun_out/fold.ncu-rep
