#!/bin/bash
# DRAM bytes read per HOPM kernel with caches NOT flushed between kernels (ncu --cache-control none):
# shows the L2 reuse between the two passes over A (TL_HOPM_KEEP_MB 64 vs 0)
mkdir -p gpurun_out
for mb in 64 0; do
  TL_HOPM_KEEP_MB=$mb timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none \
      -k regex:ttv_ -c 60 --csv --log-file gpurun_out/hopm_dram_$mb.csv python tools/experiments/hopm_keep.py > gpurun_out/hopm_dram_$mb.log 2>&1
done
