#!/bin/bash
# Run one ncu --set full capture of the kernels matching $2 driven by
# tools/ncu_drive.py $3..., then export compact CSV summaries so the
# returned gpurun_out/ stays small.  Usage: tools/ncu_box.sh NAME REGEX CFG...
set -u
name=$1; regex=$2; shift 2
timeout 300 python tools/ncu_drive.py "$@" > gpurun_out/${name}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:${regex}" -o gpurun_out/${name} python tools/ncu_drive.py "$@" > gpurun_out/${name}_ncu.log 2>&1
ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i gpurun_out/${name}.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
ncu -i gpurun_out/${name}.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>/dev/null
sz=$(stat -c %s gpurun_out/${name}.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 30000000 ]; then rm -f gpurun_out/${name}.ncu-rep; fi
gzip -f gpurun_out/${name}_source.csv gpurun_out/${name}_raw.csv 2>/dev/null
du -sh gpurun_out
