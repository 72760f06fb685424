set -u
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ttm_ -o gpurun_out/stream python tools/experiments/ncu_ttm5.py > gpurun_out/stream_ncu.log 2>&1
ncu -i gpurun_out/stream.ncu-rep --page details --csv > gpurun_out/stream_details.csv
ncu -i gpurun_out/stream.ncu-rep --page source --csv > gpurun_out/stream_source.csv; gzip -f gpurun_out/stream_source.csv
rm -f gpurun_out/stream.ncu-rep
