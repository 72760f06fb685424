mkdir -p gpurun_out
for mb in 0 96 128 160 200; do TL_TTV_KEEP_MB=$mb timeout 300 python tools/experiments/cfg2_seq.py; done 2>&1 | tee gpurun_out/cfg2_seq.txt
