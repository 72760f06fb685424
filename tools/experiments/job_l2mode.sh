# L2 policy variants: mode 1 (rest evict-first, kept normal) vs mode 2 (rest normal, kept evict-last)
mkdir -p gpurun_out
for m in 1 2; do for mb in 128 0; do TL_L2_MODE=$m TL_TTV_KEEP_MB=$mb timeout 300 python tools/experiments/cfg2_seq.py | sed "s/^/mode=$m keep=/"; done; done 2>&1 | tee gpurun_out/l2mode.txt
for m in 1 2 1 2; do TL_L2_MODE=$m timeout 200 python tools/experiments/hopm_keep.py | sed "s/^/mode=$m /"; done 2>&1 | tee -a gpurun_out/l2mode.txt
