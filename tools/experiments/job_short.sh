# short-fold path off vs on (operands >= 64 MB): representative slow cases + config-5 guards
for mb in 0 64; do echo "== TL_TTV_SHORT_MB=$mb"; TL_TTV_SHORT_MB=$mb timeout 600 python tools/experiments/ttv_cases.py; done
