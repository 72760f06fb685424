# cfg2 step GB/s vs the L2 keep budget of the public ttv (TL_TTV_KEEP_MB)
mkdir -p gpurun_out
for mb in 0 32 64 96 0 64; do
  echo -n "keep=$mb "; TL_TTV_KEEP_MB=$mb timeout 300 python bench.py --steps 10 --warmup 3 --no-components --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['mean_launch_us'])"
done 2>&1 | tee gpurun_out/ttvkeep.txt
TL_TTV_KEEP_MB=64 timeout 900 python -m pytest tests -m gpu -q -x -k "cfg2 or ttv or parity" -p no:cacheprovider 2>&1 | tail -2
