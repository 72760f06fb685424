# L2 keep rule: last k-rows (one-wave grids) vs last CTAs, HOPM and the cfg2 sequence
for r in 1 2; do for b in 0 1; do TL_KEEP_BY_CTA=$b timeout 200 python tools/experiments/hopm_keep.py | sed "s/^/by_cta=$b /"; done; done
for b in 0 1; do TL_KEEP_BY_CTA=$b timeout 300 python tools/experiments/cfg2_seq.py | sed "s/^/by_cta=$b keep=/"; done
