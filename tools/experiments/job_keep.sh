mkdir -p gpurun_out
for last in 0 1; do for mb in 48 56 64 72 80 64 0; do TL_HOPM_KEEP_LAST=$last TL_HOPM_KEEP_MB=$mb timeout 200 python tools/experiments/hopm_keep.py | sed "s/^/last=$last /"; done; done 2>&1 | tee gpurun_out/hopm_keep2.txt
