# relayout kernels: rows-copy vectors in flight x CTAs per SM (the (1,3,2,4) case), tiled transpose CTAs per SM
for u in 4 8; do for c in 4 8 16; do echo -n "rows u=$u cps=$c "; TL_COPY_ROWS_U=$u TL_COPY_ROWS_CTAS_PER_SM=$c timeout 200 python tools/experiments/copy_sweep.py; done; done
